#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_timedep.py tests/test_gpu_bdf.py -q -x -p no:cacheprovider > gpurun_out/misc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/misc_tests.log
timeout 900 python bench.py --config c4td --no-cpu > gpurun_out/misc_c4td.json 2> gpurun_out/misc_c4td.err
