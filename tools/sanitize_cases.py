"""Small launches of every kernel family for compute-sanitizer
(racecheck / memcheck / synccheck): traj_kernel on c2 (64 trajectories, one
warp, history in shared memory), c4 (8 trajectories, the register variant 22
and the TMEM variant 39), c1 with a jump log, the H(t) variant, and
bdf_kernel on c2 (16 trajectories)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_03047_b200 import configs  # noqa: E402
from paper_1810_03047_b200.engine import DeviceProblem  # noqa: E402
from paper_1810_03047_b200.problem import OdeConfig  # noqa: E402

cases = sys.argv[1:] or ["c2", "c4_22", "c4_39", "c1_log", "c4td", "bdf_c2"]
for case in cases:
    name, _, v = case.partition("_")
    if name == "bdf":
        p = configs.build(v)
        p = dataclasses.replace(p, ode=OdeConfig(method="bdf", rtol=p.ode.rtol, atol=p.ode.atol))
        n, variant, mj = 16, -1, 0
    else:
        p = configs.build(name)
        n = {"c1": 64, "c2": 64, "c4": 8, "c4td": 8}[name]
        variant = int(v) if v.isdigit() else -1
        mj = 64 if v == "log" else 0
    with DeviceProblem(p, variant=variant) as dp:
        out = dp.run(987654321, 0, n, max_jumps=mj)
    print(f"{case}: rc={out.rc} n_failed={out.n_failed} kernel {out.kernel_ms:.1f} ms", flush=True)
