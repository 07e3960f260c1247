#!/bin/bash
# A/B of alternative builds: bench lines per library tag (libqtm_<tag>.so,
# "main" = libqtm.so) for one config and kernel variant
# usage: gpu_libab.sh TAG CONFIG VARIANT LIBTAG1 [LIBTAG2 ...]
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=$1; CFG=$2; V=$3; shift 3
for rep in 1 2; do
for lt in "$@"; do
  if [ "$lt" = main ]; then L=$PWD/paper_1810_03047_b200/libqtm.so; else L=$PWD/paper_1810_03047_b200/libqtm_$lt.so; fi
  QTM_LIB=$L timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu --variant $V > gpurun_out/${TAG}_${lt}_r$rep.json 2> gpurun_out/${TAG}_${lt}_r$rep.err
done
done
