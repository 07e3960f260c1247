cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/gpu_profile.sh c2 2000 prof_c2_v5 0
