cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "oracle_identical_streams and (c2 or c1)" > gpurun_out/grp_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/grp_pytest.log
for v in 17 43 44 45 46; do
  timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --variant $v > gpurun_out/grp_c2_v$v.json 2> gpurun_out/grp_c2_v$v.err
done
