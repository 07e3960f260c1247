#!/bin/bash
# ncu capture (one launch) of the BDF kernel + source-level export
# usage: bash tools/gpu_profile_bdf.sh <config> <trajectories> <tag>
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
CFG=${1:-c3}; N=${2:-296}; TAG=${3:-bdfprof}
CMD="python bench.py --config $CFG --method bdf --trajectories $N --steps 1 --warmup 3 --no-cpu"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bdf_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_src.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
