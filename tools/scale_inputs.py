"""Measure the inputs of tools/scale_sim.py on one B200: per-trajectory attempt
counts of the full ensemble, and timed launches with one and two trajectory CTAs per SM.
    python tools/scale_inputs.py c4 39 gpurun_out/scale_inputs_c4.npz [n_total]
"""
import os, sys
import numpy as np
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
from paper_1810_03047_b200 import configs, native
from paper_1810_03047_b200.configs import N_TRAJECTORIES
from paper_1810_03047_b200.engine import DeviceProblem
from paper_1810_03047_b200.packing import pack_problem

name, variant, out_path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
n_total = int(sys.argv[4]) if len(sys.argv) > 4 else N_TRAJECTORIES[name]
pk = pack_problem(configs.build(name))
sms = 148
with DeviceProblem(pk, variant=variant) as dp:
    slots = dp.slots() if hasattr(dp, "slots") else 2 * sms
    dp.run(1, 0, 64, resident=True)
    full = dp.run(987654321, 0, n_total)
    att = full.stats[:, 0].copy()
    full_ms = min(dp.run(987654321, 0, n_total, resident=True).kernel_ms for _ in range(2))
    # one CTA per SM / two CTAs per SM: a launch of exactly that many trajectories
    alone = [dp.run(987654321, 0, sms) for _ in range(3)]
    pair = [dp.run(987654321, 0, 2 * sms) for _ in range(3)]
np.savez(out_path, attempts=att, t_full_ms=full_ms,
         t_alone_ms=min(o.kernel_ms for o in alone), work_alone=alone[0].stats[:, 0],
         t_pair_ms=min(o.kernel_ms for o in pair), work_pair=pair[0].stats[:, 0],
         grid_alone=alone[0].grid, grid_pair=pair[0].grid, grid_full=full.grid)
print(f"{name} variant {variant}: full {n_total} in {full_ms:.2f} ms (grid {full.grid}); "
      f"{sms} trajectories {min(o.kernel_ms for o in alone):.2f} ms (grid {alone[0].grid}); "
      f"{2 * sms} trajectories {min(o.kernel_ms for o in pair):.2f} ms (grid {pair[0].grid})")
