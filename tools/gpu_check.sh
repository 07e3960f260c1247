#!/bin/bash
# one GPU-box session: smoke, GPU tests, bench lines (see gpurun_out/)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu >> gpurun_out/bench_all.log 2>&1
done
timeout 600 python bench.py --config c5 --trajectories 2000 --steps 1 --warmup 3 --no-cpu >> gpurun_out/bench_all.log 2>&1
echo "bench_all done" >> gpurun_out/bench_all.log
