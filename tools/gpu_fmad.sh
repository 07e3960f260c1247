#!/bin/bash
# the fused-multiply-add build (libqtm_fmad.so): c4 A/B of variants 22/39 and the whole GPU suite
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
export QTM_LIB=$PWD/paper_1810_03047_b200/libqtm_fmad.so
for v in 22 39; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --variant $v > gpurun_out/fm_c4_v$v.json 2> gpurun_out/fm_c4_v$v.err
done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/fm_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fm_pytest.log
