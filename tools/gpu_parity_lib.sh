#!/bin/bash
# the GPU suite and the c4 bench line under the unfused parity library (QTM_FMAD=0 build)
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
L=$PWD/paper_1810_03047_b200/libqtm_parity.so
QTM_LIB=$L timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/parity_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/parity_pytest_gpu.log
QTM_LIB=$L timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/parity_bench_c4.json 2> gpurun_out/parity_bench_c4.err
