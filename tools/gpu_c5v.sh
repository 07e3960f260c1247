#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python tools/ab_time.py c5:8192:27 c5:8192:39 > gpurun_out/c5v_abtime.txt 2>&1
bash tools/gpu_ncu.sh c5v_c5_full c5 2048 39
python tools/summarize_ncu.py gpurun_out/c5v_c5_full gpurun_out/c5v_c5_full_sum > gpurun_out/c5v_c5_full_sum.log 2>&1
rm -f gpurun_out/c5v_c5_full.ncu-rep gpurun_out/c5v_c5_full_src.csv gpurun_out/c5v_c5_full_cuda.csv
