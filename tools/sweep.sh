#!/bin/bash
# kernel-variant sweep: one bench line per (config, variant)
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
OUT=gpurun_out/sweep.log; : > $OUT
run() { timeout 300 python bench.py --config $1 --variant $2 --steps 1 --warmup 3 --no-cpu $3 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$1', 'variant', $2, d['config']['kernel_variant'], 'grid', d['config']['grid_ctas'], 'value %.0f'%d['value'], 'kernel_ms %.1f'%r['kernel_ms'], 'frac %.3f'%r['frac'])" >> $OUT 2>&1; }
for v in 6 7 9; do run c4 $v; done
for v in 6 8 14 15 16 7; do run c5 $v "--trajectories 2000"; done
for v in 0 10 11; do run c2 $v; done
for v in 2 3 12 13; do run c3 $v; done
for v in 0 10; do run c1 $v; done
