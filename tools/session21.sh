cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/ab_run.sh "c2:5000:0 c3:4000:2 c4:4096:6 c5:600:15" libqtm_rcp.so libqtm_sq.so
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
