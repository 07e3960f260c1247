cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for c in c4 c2 c3; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/s4_$c.json 2>&1; done
timeout 300 python bench.py --config c5 --trajectories 2000 --steps 1 --warmup 3 --no-cpu > gpurun_out/s4_c5.json 2>&1
bash tools/gpu_profile.sh c2 1000 prof_c2_v3
bash tools/gpu_profile.sh c5 200 prof_c5_v3
bash tools/gpu_profile.sh c4 512 prof_c4_v3
