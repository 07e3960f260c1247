cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for lt in main m5 m6; do
  if [ "$lt" = main ]; then L=$PWD/paper_1810_03047_b200/libqtm.so; else L=$PWD/paper_1810_03047_b200/libqtm_$lt.so; fi
  QTM_LIB=$L timeout 900 python bench.py --config c3 --method bdf --steps 1 --warmup 3 --no-cpu > gpurun_out/b5_$lt.json 2> gpurun_out/b5_$lt.err
done
