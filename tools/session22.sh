cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/ab_run.sh "c2:5000:0 c3:4000:2 c4:4096:6 c5:600:15" libqtm_base.so libqtm_ih.so
timeout 600 python tools/phases.py c4:1024:6 c5:300:15 c2:2000:0 c3:2000:2 > gpurun_out/phases.txt 2>&1
