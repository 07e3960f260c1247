cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
export QTM_LIB=$PWD/paper_1810_03047_b200/libqtm_b128.so
for nt in 64 128; do
QTM_BDF_HBM=1 QTM_BDF_THREADS=$nt timeout 900 python bench.py --config c3 --method bdf --steps 1 --warmup 3 --no-cpu > gpurun_out/b2_hbm$nt.json 2> gpurun_out/b2_hbm$nt.err
done
QTM_BDF_HBM=1 QTM_BDF_THREADS=64 timeout 900 python bench.py --config c2 --method bdf --steps 1 --warmup 3 --no-cpu > gpurun_out/b2_c2hbm64.json 2> gpurun_out/b2_c2hbm64.err
timeout 900 python bench.py --config c2 --method bdf --steps 1 --warmup 3 --no-cpu > gpurun_out/b2_c2base.json 2> gpurun_out/b2_c2base.err
