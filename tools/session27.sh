cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/gpu_profile.sh c4 1024 p27_c4_v6 6
bash tools/gpu_profile.sh c4 1024 p27_c4_v22 22
for t in p27_c4_v6 p27_c4_v22; do
  ncu -i gpurun_out/$t.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${t}_src.csv 2>/dev/null
  ncu -i gpurun_out/$t.ncu-rep --page raw --csv > gpurun_out/${t}_raw.csv 2>/dev/null
done
