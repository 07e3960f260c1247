#!/bin/bash
# BDF capture: bench lines (device + CPU oracle leg), reference arm, ncu of bdf_kernel
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=${1:-r03}
for c in c1 c2; do
  timeout 900 python bench.py --config $c --method bdf > gpurun_out/${TAG}_bench_bdf_$c.json 2> gpurun_out/${TAG}_bench_bdf_$c.err
done
timeout 1200 python bench.py --config c3 --method bdf --steps 1 --warmup 3 > gpurun_out/${TAG}_bench_bdf_c3.json 2> gpurun_out/${TAG}_bench_bdf_c3.err
timeout 900 python bench.py --impl reference --config c3 --method bdf --steps 1 --warmup 0 > gpurun_out/${TAG}_bench_bdf_ref_c3.json 2> gpurun_out/${TAG}_bench_bdf_ref_c3.err
bash tools/gpu_profile_bdf.sh c3 1000 ${TAG}_bdf_c3
ncu -i gpurun_out/${TAG}_bdf_c3.ncu-rep --page raw --csv > gpurun_out/${TAG}_bdf_c3_raw.csv 2>/dev/null
