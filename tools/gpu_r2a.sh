#!/bin/bash
# round 2: new parity tests at reference scale, drop-in types, self-launched ranks
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_scale.py tests/test_gpu_dropin.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "scale or dropin or reference_problem or odefailure or block_partials or failures" > gpurun_out/r2a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu > gpurun_out/r2a_bench2.json 2> gpurun_out/r2a_bench2.err
echo "bench2 rc=$?" >> gpurun_out/r2a_bench2.err
