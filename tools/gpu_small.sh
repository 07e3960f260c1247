#!/bin/bash
# one-thread-per-trajectory kernel: parity subset + c1 bench per variant
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider -k "c1 or recording or scenarios or forced or max_steps or no_support or rabi or drop_in" > gpurun_out/sm_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/sm_pytest.log
for v in 0 40 41 42 43; do
  timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --variant $v > gpurun_out/sm_c1_v$v.json 2> gpurun_out/sm_c1_v$v.err
done
