#!/bin/bash
# GPU suite + short-config bench lines (run_impl changes)
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/rt_bench.log
for c in c1 c2 c4; do timeout 600 python bench.py --config $c --no-cpu >> gpurun_out/rt_bench.log 2>&1; done
