"""One short BDF run of c5 (t in [0, 2]) for an ncu capture of bdf_kernel."""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_03047_b200 import configs
from paper_1810_03047_b200.engine import DeviceProblem, stats_dict
from paper_1810_03047_b200.packing import pack_problem
from paper_1810_03047_b200.problem import OdeConfig
p = configs.build(sys.argv[1] if len(sys.argv) > 1 else "c5")
p = dataclasses.replace(p, t_to=2.0, n_steps=20, ode=OdeConfig(method="bdf", rtol=p.ode.rtol, atol=p.ode.atol))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 148
with DeviceProblem(pack_problem(p)) as dp:
    for _ in range(2):
        out = dp.run(987654321, 0, n, resident=True)
    print("kernel_ms", out.kernel_ms, stats_dict(out.stats_total))
