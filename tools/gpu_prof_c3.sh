#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/gpu_profile.sh c3 20000 p_c3 12
ncu -i gpurun_out/p_c3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/p_c3_src.csv 2>/dev/null
ncu -i gpurun_out/p_c3.ncu-rep --page details --csv > gpurun_out/p_c3_details.csv 2>/dev/null
rm -f gpurun_out/p_c3.ncu-rep
