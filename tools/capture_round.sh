#!/bin/bash
# Round capture (B200_PROFILING.md recipe): bench lines for every config and
# both arms, the ncu launch list of the default c4 command, and one
# --set full capture of the trajectory kernel (c4; c5 on a 2048-trajectory
# sample).  usage: bash tools/capture_round.sh <tag> [c4 variant] [c5 variant]
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=${1:-r01}; V4=${2:-22}; V5=${3:-27}
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 1800 python bench.py --config c5 --steps 1 --warmup 3 > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 900 python bench.py --config c4td > gpurun_out/${TAG}_bench_c4td.json 2> gpurun_out/${TAG}_bench_c4td.err
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
CMD="python bench.py --steps 2 --warmup 3 --variant $V4 --no-cpu"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c4_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_launches.log
$CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 3 -c 1 -o gpurun_out/${TAG}_c4_full $CMD > gpurun_out/${TAG}_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_full.log
C5="python bench.py --config c5 --trajectories 2048 --steps 1 --warmup 3 --variant $V5 --no-cpu"
$C5 > gpurun_out/${TAG}_c5plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 3 -c 1 -o gpurun_out/${TAG}_c5_full $C5 > gpurun_out/${TAG}_c5full.log 2>&1
echo "c5 full rc=$?" >> gpurun_out/${TAG}_c5full.log
for k in c4 c5; do
  if [ -f gpurun_out/${TAG}_${k}_full.ncu-rep ]; then
    ncu -i gpurun_out/${TAG}_${k}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_${k}_raw.csv 2>/dev/null
    ncu -i gpurun_out/${TAG}_${k}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_${k}_details.csv 2>/dev/null
    ncu -i gpurun_out/${TAG}_${k}_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_${k}_src.csv 2>/dev/null
  fi
done
