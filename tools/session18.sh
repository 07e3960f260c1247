cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 600 python tools/phases.py c4:1024:6 c5:300:15 c2:2000:0 c3:2000:2 > gpurun_out/phases.txt 2>&1
