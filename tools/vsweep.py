"""Time every candidate kernel variant on one config (resident inputs).

    python tools/vsweep.py c4 [n_trajectories] [variant ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_03047_b200 import configs, native  # noqa: E402
from paper_1810_03047_b200.engine import DeviceProblem, candidate_variants  # noqa: E402
from paper_1810_03047_b200.packing import pack_problem  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else configs.N_TRAJECTORIES[name]
pk = pack_problem(configs.build(name))
vs = [int(v) for v in sys.argv[3:]] or candidate_variants(pk.dim)
table = native.variants()
for v in vs:
    with DeviceProblem(pk, variant=v) as dp:
        dp.run(987654321, 0, min(n, 512), resident=True)
        out = dp.run(987654321, 0, n, resident=True)
        print(f"{name} v{v} {table[v]} grid {out.grid} kernel_ms {out.kernel_ms:.2f} "
              f"traj/s {n / out.kernel_ms * 1e3:.0f} {dp.layout()} ovf_steps {out.stats_total[13]}",
              flush=True)
