cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/gpu_libab.sh lab7 c4 39 main fw
for lt in main fw; do
  if [ "$lt" = main ]; then L=$PWD/paper_1810_03047_b200/libqtm.so; else L=$PWD/paper_1810_03047_b200/libqtm_$lt.so; fi
  QTM_LIB=$L timeout 900 python bench.py --config c5 --trajectories 8192 --steps 2 --warmup 3 --no-cpu --variant 27 > gpurun_out/lab7c5_${lt}_r1.json 2> gpurun_out/lab7c5_${lt}_r1.err
done
QTM_LIB=$PWD/paper_1810_03047_b200/libqtm_fw.so timeout 1500 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "identical" > gpurun_out/ab7_fw_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab7_fw_pytest.log
