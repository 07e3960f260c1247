#!/bin/bash
# Round capture: default bench line, ncu launch list and one --set full
# capture of the trajectory kernel for the same command (B200_PROFILING.md).
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=${1:-r01}
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
CMD="python bench.py --steps 2 --warmup 3 --variant 6 --no-cpu"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_launches.log
$CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 3 -c 1 -o gpurun_out/${TAG}_c4_full $CMD > gpurun_out/${TAG}_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_full.log
