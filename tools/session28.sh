cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/vsweep.py c4 4096 6 22 > gpurun_out/s28.txt 2>&1
timeout 600 python tools/vsweep.py c5 8192 15 >> gpurun_out/s28.txt 2>&1
timeout 600 python tools/vsweep.py c3 20000 >> gpurun_out/s28.txt 2>&1
timeout 600 python tools/vsweep.py c2 5000 17 >> gpurun_out/s28.txt 2>&1
