cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for m in off nvml smi nvml; do
  QTM_CLOCKS=$m timeout 600 python bench.py --variant 6 --no-cpu --steps 4 > gpurun_out/clk_$m.json 2>&1
  echo "mode $m" >> gpurun_out/clk_summary.txt
  python -c "import json; d=json.loads(open('gpurun_out/clk_$m.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['step_ms'], d['roofline']['kernel_ms'], d['clocks'])" >> gpurun_out/clk_summary.txt 2>&1
done
