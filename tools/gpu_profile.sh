#!/bin/bash
# ncu capture of the trajectory kernel (one launch) for a config
# usage: bash tools/gpu_profile.sh <config> <trajectories> <tag>
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
CFG=${1:-c4}; NT=${2:-1024}; TAG=${3:-prof}
CMD="python bench.py --config $CFG --trajectories $NT --steps 1 --warmup 3 --no-cpu ${4:+--variant $4}"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
