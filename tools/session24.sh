cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/ab_run.sh "c1:500:0 c1:500:17 c2:5000:0 c2:5000:17 c3:4000:2 c3:4000:19 c3:4000:20 c3:4000:12" libqtm.so
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
