#!/bin/bash
# Final capture of a round: bench lines for every config and method, the
# reference arm, the GPU suite and smoke; ncu launch list of the default c4
# command.  usage: bash tools/capture_final.sh <tag>
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
TAG=${1:-r04}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
for c in c1 c2 c3 c4 c4td; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 1800 python bench.py --config c5 --steps 1 --warmup 3 > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
for c in c1 c2; do
  timeout 900 python bench.py --config $c --method bdf > gpurun_out/${TAG}_bench_bdf_$c.json 2> gpurun_out/${TAG}_bench_bdf_$c.err
done
timeout 1200 python bench.py --config c3 --method bdf --steps 1 --warmup 3 > gpurun_out/${TAG}_bench_bdf_c3.json 2> gpurun_out/${TAG}_bench_bdf_c3.err
CMD="python bench.py --steps 2 --warmup 3 --variant 22 --no-cpu"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c4_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
