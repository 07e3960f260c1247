cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 600 python tools/phases.py c2:2000:0 c4:1024:6 > gpurun_out/phases.txt 2>&1
