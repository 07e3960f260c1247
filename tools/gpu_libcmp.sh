#!/bin/bash
# A/B of a tagged library against libqtm.so: bitwise comparison of the
# per-trajectory outputs on several configs / variants, then bench lines,
# then (optionally) the GPU suite under the tagged library.
# usage: gpu_libcmp.sh TAG LIBTAG [suite]   (libqtm_LIBTAG.so against libqtm.so)
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=$1; LT=$2
P=$PWD/paper_1810_03047_b200
SPECS="c4:296:39 c4:148:22 c5:128:27 c3:512:12 c2:512:17 c1:500:0 c4td:148:36 c4:128:6 c5:64:26 c4:64:38 c3:512:3 c3:256:13 c2:512:1 c2:512:0"
QTM_LIB=$P/libqtm.so timeout 900 python tools/lib_dump.py dump gpurun_out/${TAG}_base.npz $SPECS > gpurun_out/${TAG}_dump_base.log 2>&1
QTM_LIB=$P/libqtm_$LT.so timeout 900 python tools/lib_dump.py dump gpurun_out/${TAG}_new.npz $SPECS > gpurun_out/${TAG}_dump_new.log 2>&1
python tools/lib_dump.py cmp gpurun_out/${TAG}_base.npz gpurun_out/${TAG}_new.npz > gpurun_out/${TAG}_cmp.log 2>&1
rm -f gpurun_out/${TAG}_base.npz gpurun_out/${TAG}_new.npz
for rep in 1 2; do
for lt in main $LT; do
  if [ "$lt" = main ]; then L=$P/libqtm.so; else L=$P/libqtm_$lt.so; fi
  QTM_LIB=$L timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_c4_${lt}_r$rep.json 2> gpurun_out/${TAG}_c4_${lt}_r$rep.err
done
done
rm -f gpurun_out/${TAG}_abtime.txt
for lt in main $LT; do
  if [ "$lt" = main ]; then L=$P/libqtm.so; else L=$P/libqtm_$lt.so; fi
  QTM_LIB=$L timeout 900 python tools/ab_time.py c5:4096:27 c3:20000:12 c2:5000:17 c4td:4096:36 >> gpurun_out/${TAG}_abtime.txt 2>&1
done
if [ "$3" = suite ]; then
  QTM_LIB=$P/libqtm_$LT.so timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
fi
