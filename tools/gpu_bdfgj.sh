cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bdf.py -m gpu -q -p no:cacheprovider > gpurun_out/gj_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gj_pytest.log
for m in gj inv; do
  QTM_BDF_SOLVE=$m timeout 900 python bench.py --config c3 --method bdf --steps 1 --warmup 3 --no-cpu > gpurun_out/gj_c3_$m.json 2> gpurun_out/gj_c3_$m.err
done
