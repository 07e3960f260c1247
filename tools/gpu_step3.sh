#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
P=$PWD/paper_1810_03047_b200
timeout 600 python tools/scale_inputs.py c4 39 gpurun_out/scale_inputs_c4.npz > gpurun_out/scale_inputs_c4.log 2>&1
for rep in 1 2; do
for lt in main pk pk1; do
  if [ "$lt" = main ]; then L=$P/libqtm.so; else L=$P/libqtm_$lt.so; fi
  QTM_LIB=$L timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu > gpurun_out/s3_c4_${lt}_r$rep.json 2> gpurun_out/s3_c4_${lt}_r$rep.err
done
done
rm -f gpurun_out/s3_abtime.txt
for lt in main pk pk1; do
  if [ "$lt" = main ]; then L=$P/libqtm.so; else L=$P/libqtm_$lt.so; fi
  QTM_LIB=$L timeout 900 python tools/ab_time.py c5:4096:27 c3:20000:12 c2:5000:17 c4td:4096:36 >> gpurun_out/s3_abtime.txt 2>&1
done
