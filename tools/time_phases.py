"""Time the phases of one public-API call (create / run / destroy) per config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_03047_b200 import configs
from paper_1810_03047_b200.configs import N_TRAJECTORIES
from paper_1810_03047_b200.engine import DeviceProblem
from paper_1810_03047_b200.packing import pack_problem

for name in sys.argv[1:] or ["c1", "c2", "c4"]:
    pk = pack_problem(configs.build(name))
    n = N_TRAJECTORIES[name] if name != "c5" else 500
    for rep in range(3):
        t0 = time.perf_counter()
        dp = DeviceProblem(pk)
        t1 = time.perf_counter()
        out = dp.run(987654321, 0, n, resident=True)
        t2 = time.perf_counter()
        out2 = dp.run(987654321, 0, n, resident=True)
        t3 = time.perf_counter()
        dp.close()
        t4 = time.perf_counter()
        print(f"{name} rep{rep}: create {1e3*(t1-t0):.1f} ms  run1 {1e3*(t2-t1):.1f} ms (kernel {out.kernel_ms:.1f}, total {out.total_ms:.1f})  "
              f"run2 {1e3*(t3-t2):.1f} ms (kernel {out2.kernel_ms:.1f})  destroy {1e3*(t4-t3):.1f} ms", flush=True)
