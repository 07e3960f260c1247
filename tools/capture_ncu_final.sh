#!/bin/bash
# --set full captures of the trajectory kernel (c4 and a c5 sample) for a tag
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=${1:-r05}
CMD="python bench.py --steps 2 --warmup 3 --variant 22 --no-cpu"
$CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 3 -c 1 -o gpurun_out/${TAG}_c4_full $CMD > gpurun_out/${TAG}_full.log 2>&1
C5="python bench.py --config c5 --trajectories 2048 --steps 1 --warmup 3 --variant 27 --no-cpu"
$C5 > gpurun_out/${TAG}_c5plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 3 -c 1 -o gpurun_out/${TAG}_c5_full $C5 > gpurun_out/${TAG}_c5full.log 2>&1
for k in c4 c5; do
  if [ -f gpurun_out/${TAG}_${k}_full.ncu-rep ]; then
    ncu -i gpurun_out/${TAG}_${k}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_${k}_raw.csv 2>/dev/null
    ncu -i gpurun_out/${TAG}_${k}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_${k}_details.csv 2>/dev/null
    ncu -i gpurun_out/${TAG}_${k}_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_${k}_src.csv 2>/dev/null
    rm -f gpurun_out/${TAG}_${k}_full.ncu-rep
  fi
done
