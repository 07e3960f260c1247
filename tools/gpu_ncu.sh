#!/bin/bash
# ncu --set full capture of one trajectory-kernel launch + exports
# usage: bash tools/gpu_ncu.sh TAG CONFIG TRAJECTORIES [VARIANT]
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=$1; CFG=${2:-c4}; NT=${3:-1184}; V=$4
CMD="python bench.py --config $CFG --trajectories $NT --steps 1 --warmup 3 --no-cpu ${V:+--variant $V}"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"traj_kernel|traj1_kernel" -s 3 -c 1 \
    -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
if [ -f gpurun_out/${TAG}.ncu-rep ]; then
  ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_src.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source cuda > gpurun_out/${TAG}_cuda.csv 2>/dev/null
fi
