#!/bin/bash
# Round capture (B200_PROFILING.md recipe): bench lines for every config and
# both arms, the GPU suite and smoke, per-shard times of the multi-GPU split,
# the ncu launch list of the default c4 command, and one --set full capture of
# the trajectory kernel (c4; c5 on a 2048-trajectory sample), summarised on the
# box (the .ncu-rep files stay there).
# usage: bash tools/capture_round.sh <tag> [c4 variant] [c5 variant]
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=${1:-r2}; V4=${2:-39}; V5=${3:-27}
for c in c1 c2 c3 c4 c4td; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c --method bdf > gpurun_out/${TAG}_bench_bdf_$c.json 2> gpurun_out/${TAG}_bench_bdf_$c.err
done
timeout 1800 python bench.py --config c5 --steps 1 --warmup 3 > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 600 python bench.py --gpus 2 --steps 3 --no-cpu > gpurun_out/${TAG}_bench_gpus2.json 2> gpurun_out/${TAG}_bench_gpus2.err
timeout 900 python tools/shard_times.py c4 $V4 > gpurun_out/${TAG}_shard_times_c4.json 2> gpurun_out/${TAG}_shard_times_c4.err
QTM_ORDER=0 timeout 900 python tools/shard_times.py c4 $V4 > gpurun_out/${TAG}_shard_times_c4_index_order.json 2> gpurun_out/${TAG}_shard_times_c4_index_order.err
timeout 600 python tools/scale_inputs.py c4 $V4 gpurun_out/${TAG}_scale_inputs_c4.npz > gpurun_out/${TAG}_scale_inputs_c4.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
CMD="python bench.py --steps 2 --warmup 3 --variant $V4 --no-cpu"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c4_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_launches.log
bash tools/gpu_ncu.sh ${TAG}_c4_full c4 4096 $V4
bash tools/gpu_ncu.sh ${TAG}_c5_full c5 2048 $V5
for t in ${TAG}_c4_full ${TAG}_c5_full; do
  python tools/summarize_ncu.py gpurun_out/$t gpurun_out/${t}_sum > gpurun_out/${t}_sum.log 2>&1
  rm -f gpurun_out/$t.ncu-rep gpurun_out/${t}_src.csv gpurun_out/${t}_cuda.csv
done
