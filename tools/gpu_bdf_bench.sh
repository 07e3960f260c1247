#!/bin/bash
# BDF bench lines (exploration): c1/c2 full size, c3 on a sample
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for c in c1 c2; do
  timeout 600 python bench.py --config $c --method bdf --steps 2 --warmup 3 --no-cpu >> gpurun_out/bdf_bench.log 2>&1
done
timeout 900 python bench.py --config c3 --method bdf --trajectories 2000 --steps 1 --warmup 3 --no-cpu >> gpurun_out/bdf_bench.log 2>&1
timeout 900 python bench.py --config c4 --method bdf --trajectories 148 --steps 1 --warmup 3 --no-cpu >> gpurun_out/bdf_bench.log 2>&1
echo done >> gpurun_out/bdf_bench.log
