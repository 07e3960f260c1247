#!/bin/bash
# A/B: exact (fmad=false) vs fma library on the same box
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 300 python tools/time_phases.py c1 c2 c4 > gpurun_out/phases.log 2>&1
for lib in libqtm.so libqtm_fma.so; do
  for c in c4 c2 c3; do
    QTM_LIB=$PWD/paper_1810_03047_b200/$lib timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/ab_${lib}_$c.json 2>&1
  done
  QTM_LIB=$PWD/paper_1810_03047_b200/$lib timeout 300 python bench.py --config c5 --trajectories 2000 --steps 1 --warmup 3 --no-cpu > gpurun_out/ab_${lib}_c5.json 2>&1
done
QTM_LIB=$PWD/paper_1810_03047_b200/libqtm_fma.so timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_fma.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
