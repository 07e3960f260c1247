#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/ab.txt
bash tools/ab_run.sh "c4:4096:22 c5:2048:27 c3:20000:12 c2:5000:17" libqtm_base.so libqtm.so libqtm_base.so libqtm.so
