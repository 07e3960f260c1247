cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bdf.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider -k "bdf" > gpurun_out/b3_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/b3_pytest.log
for c in c1 c2 c3; do timeout 900 python bench.py --config $c --method bdf > gpurun_out/b3_bdf_$c.json 2> gpurun_out/b3_bdf_$c.err; done
