"""Largest difference between two kernel variants' per-trajectory outputs on the
same streams (jump logs must be equal): python tools/cmp_variants.py c4td 150 36 43"""
import os, sys
import numpy as np
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
from paper_1810_03047_b200 import configs
from paper_1810_03047_b200.engine import DeviceProblem, run_logged
from paper_1810_03047_b200.packing import pack_problem

name, n, va, vb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
pk = pack_problem(configs.build(name))
outs = []
for v in (va, vb):
    with DeviceProblem(pk, variant=v) as dp:
        outs.append(run_logged(dp, 987654321, 0, n))
        print(f"variant {v}: resident CTAs {dp.max_resident()}, kernel {outs[-1].kernel_ms:.2f} ms")
a, b = outs
print("jump counts equal:", np.array_equal(a.jump_count, b.jump_count),
      "| status equal:", np.array_equal(a.status, b.status),
      "| max |dvalue|:", float(np.abs(a.values - b.values).max()),
      "| bitwise:", np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64)))
