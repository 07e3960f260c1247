cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1500 python bench.py --config c5 --steps 1 --warmup 3 > gpurun_out/s26_c5.json 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/s26_c4.json 2>&1
