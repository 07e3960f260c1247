#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/gpu_profile_bdf.sh c1 500 pbc1
python tools/src_hot.py gpurun_out/pbc1_src.csv 30 > gpurun_out/pbc1_hot.txt 2>&1
rm -f gpurun_out/pbc1.ncu-rep gpurun_out/pbc1_src.csv
