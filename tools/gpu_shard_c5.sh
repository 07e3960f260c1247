#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
SHARD_REPS=1 timeout 1500 python tools/shard_times.py c5 39 > gpurun_out/shard_times_c5.json 2> gpurun_out/shard_times_c5.err
timeout 600 python -m pytest tests/test_gpu_order.py -m gpu -q -s -p no:cacheprovider > gpurun_out/order_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/order_test.log
