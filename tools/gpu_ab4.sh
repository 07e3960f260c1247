cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --variant 39 > gpurun_out/ab4_c4_v39.json 2> gpurun_out/ab4_c4_v39.err
for v in 27 39; do
timeout 900 python bench.py --config c5 --trajectories 8192 --steps 2 --warmup 3 --no-cpu --variant $v > gpurun_out/ab4_c5_v$v.json 2> gpurun_out/ab4_c5_v$v.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "oracle_identical_streams and (c4 or c5)" > gpurun_out/ab4_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab4_pytest.log
