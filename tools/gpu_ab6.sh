cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/gpu_libab.sh lab6 c4 39 main cmac
for v in 36 40; do
  timeout 600 python bench.py --config c4td --steps 5 --warmup 3 --no-cpu --variant $v > gpurun_out/ab6_c4td_v$v.json 2> gpurun_out/ab6_c4td_v$v.err
done
timeout 900 python -m pytest tests/test_gpu_timedep.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider > gpurun_out/ab6_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab6_pytest.log
QTM_LIB=$PWD/paper_1810_03047_b200/libqtm_cmac.so timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "identical" > gpurun_out/ab6_cmac_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab6_cmac_pytest.log
