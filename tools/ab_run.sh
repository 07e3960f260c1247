#!/bin/bash
# usage: bash tools/ab_run.sh "<specs>" lib1 lib2 ...
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
SPECS=$1; shift
for lib in "$@"; do
  QTM_LIB=$PWD/paper_1810_03047_b200/$lib timeout 900 python tools/ab_time.py $SPECS >> gpurun_out/ab.txt 2>&1
done
