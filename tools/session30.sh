cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
T=p30_c5_v15
bash tools/gpu_profile.sh c5 1184 $T 15
ncu -i gpurun_out/$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_src.csv 2>/dev/null
ncu -i gpurun_out/$T.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null
rm -f gpurun_out/$T.ncu-rep
