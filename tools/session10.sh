cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu > gpurun_out/def1.json 2>&1
timeout 600 python bench.py --no-cpu --steps 5 > gpurun_out/def2.json 2>&1
