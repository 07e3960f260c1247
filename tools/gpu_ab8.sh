cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
bash tools/gpu_libab.sh lab8 c4 39 main cw
QTM_LIB=$PWD/paper_1810_03047_b200/libqtm_cw.so timeout 1500 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -s -p no:cacheprovider -k "identical and c4" > gpurun_out/ab8_cw_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab8_cw_pytest.log
