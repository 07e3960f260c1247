cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/phases.py c4:1024:6 c5:300:15 c2:2000:0 c3:2000:2 > gpurun_out/phases.txt 2>&1
bash tools/sweep.sh
