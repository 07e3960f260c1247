#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
python tools/prof_bdf_c5.py c5 148 > gpurun_out/pb5_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bdf_kernel -s 1 -c 1 -o gpurun_out/pb5 python tools/prof_bdf_c5.py c5 148 > gpurun_out/pb5_ncu.log 2>&1
ncu -i gpurun_out/pb5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pb5_src.csv 2>/dev/null
rm -f gpurun_out/pb5.ncu-rep
