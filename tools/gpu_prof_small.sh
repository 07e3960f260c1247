#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for spec in "c1 500 p_c1" "c2 5000 p_c2"; do
  set -- $spec
  bash tools/gpu_profile.sh $1 $2 $3
  ncu -i gpurun_out/$3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$3_src.csv 2>/dev/null
  ncu -i gpurun_out/$3.ncu-rep --page details --csv > gpurun_out/$3_details.csv 2>/dev/null
  rm -f gpurun_out/$3.ncu-rep
done
