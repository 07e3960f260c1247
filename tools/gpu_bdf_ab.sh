#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bdf.py -q -x -p no:cacheprovider > gpurun_out/bdf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bdf_tests.log
QTM_BDF_SOLVE=lu timeout 900 python -m pytest tests/test_gpu_bdf.py -q -x -p no:cacheprovider >> gpurun_out/bdf_tests.log 2>&1; echo "lu rc=$?" >> gpurun_out/bdf_tests.log
for s in inv lu; do
  QTM_BDF_SOLVE=$s timeout 900 python bench.py --config c3 --method bdf --trajectories 1000 --steps 1 --warmup 3 --no-cpu >> gpurun_out/bdf_ab.log 2>&1
  QTM_BDF_SOLVE=$s timeout 900 python bench.py --config c2 --method bdf --steps 2 --warmup 3 --no-cpu >> gpurun_out/bdf_ab.log 2>&1
done
