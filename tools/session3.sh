cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 300 python tools/time_phases.py c1 c2 c3 c4 > gpurun_out/phases.log 2>&1
bash tools/gpu_profile.sh c4 1024 prof_c4_v2
