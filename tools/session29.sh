cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
T=${1:-p29_c4_v22}; V=${2:-22}
bash tools/gpu_profile.sh c4 1024 $T $V
ncu -i gpurun_out/$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_src.csv 2>/dev/null
ncu -i gpurun_out/$T.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null
rm -f gpurun_out/$T.ncu-rep
