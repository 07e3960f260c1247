#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/gpu_pk.sh s5 base
timeout 900 python tools/shard_times.py c4 39 > gpurun_out/s5_shard_times_c4.json 2> gpurun_out/s5_shard_times_c4.err
QTM_ORDER=0 timeout 900 python tools/shard_times.py c4 39 > gpurun_out/s5_shard_times_c4_noorder.json 2> gpurun_out/s5_shard_times_c4_noorder.err
