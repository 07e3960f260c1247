cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/gpu_profile.sh c5 200 prof_c5_v4 15
bash tools/gpu_profile.sh c4 512 prof_c4_v4 6
bash tools/gpu_profile.sh c2 1000 prof_c2_v4 0
