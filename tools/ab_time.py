"""Kernel time of each config under the library in $QTM_LIB (A/B helper)."""
import os, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
from paper_1810_03047_b200 import configs, native
from paper_1810_03047_b200.engine import DeviceProblem
from paper_1810_03047_b200.packing import pack_problem

lib = os.path.basename(os.environ.get("QTM_LIB", "libqtm.so"))
for spec in sys.argv[1:]:
    name, n, v = (spec.split(":") + ["-1"])[:3]
    pk = pack_problem(configs.build(name))
    with DeviceProblem(pk, variant=int(v)) as dp:
        dp.run(1, 0, min(int(n), 256), resident=True)
        outs = [dp.run(987654321, 0, int(n), resident=True) for _ in range(2)]
    ts = [o.kernel_ms for o in outs]
    print(f"{lib:18s} {name} n={n} v={native.variants()[int(v)] if int(v) >= 0 else 'auto'} "
          f"kernel_ms {min(ts):9.2f} attempts {int(outs[0].stats_total[0])}", flush=True)
