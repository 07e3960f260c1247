#!/bin/bash
# round 2: TMEM variant (39) parity + A/B against the register variant (22) on c4
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "oracle_identical_streams and c4" > gpurun_out/r2b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
for v in 22 39; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --variant $v > gpurun_out/r2b_bench_v$v.json 2> gpurun_out/r2b_bench_v$v.err
done
timeout 1200 python -m pytest tests/test_gpu_scale.py -m gpu -q -s -p no:cacheprovider -k identical > gpurun_out/r2b_scale.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_scale.log
