cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu > gpurun_out/c5_full.json 2>&1
timeout 600 python bench.py > gpurun_out/c4_default.json 2>&1
