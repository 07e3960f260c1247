#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_order.py -m gpu -q -s -p no:cacheprovider > gpurun_out/s4_order_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4_order_test.log
for rep in 1 2; do
for o in 0 1; do
  QTM_ORDER=$o timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu > gpurun_out/s4_c4_order${o}_r$rep.json 2> gpurun_out/s4_c4_order${o}_r$rep.err
done
done
rm -f gpurun_out/s4_abtime.txt
for o in 0 1; do
  echo "QTM_ORDER=$o" >> gpurun_out/s4_abtime.txt
  QTM_ORDER=$o timeout 900 python tools/ab_time.py c5:4096:27 c3:20000:12 c2:5000:17 c4td:4096:36 c4:512:39 c4:1024:39 c4:2048:39 >> gpurun_out/s4_abtime.txt 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/s4_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4_pytest_gpu.log
