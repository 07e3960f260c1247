"""Per-phase cycle breakdown of the attempt loop (needs libqtm_phases.so:
QTM_PHASES=1 QTM_BUILD_TAG=phases python -m paper_1810_03047_b200.build)."""
import os, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("QTM_LIB", os.path.join(HERE, "paper_1810_03047_b200", "libqtm_phases.so"))
sys.path.insert(0, HERE)
from paper_1810_03047_b200 import configs, native
from paper_1810_03047_b200.engine import DeviceProblem, stats_dict
from paper_1810_03047_b200.packing import pack_problem

for spec in sys.argv[1:] or ["c4:512:6"]:
    name, n, v = (spec.split(":") + ["-1"])[:3]
    pk = pack_problem(configs.build(name))
    with DeviceProblem(pk, variant=int(v)) as dp:
        dp.run(1, 0, min(int(n), 64), resident=True)
        out = dp.run(987654321, 0, int(n), resident=True)
    ph = native.phase_cycles()
    st = stats_dict(out.stats_total)
    tot = sum(ph.values())
    print(f"== {name} n={n} variant={native.variants()[out.variant]} kernel {out.kernel_ms:.1f} ms, "
          f"attempts {st['attempts']}, corr iters {st['corr_iters']}")
    for k, c in ph.items():
        print(f"   {k:24s} {100 * c / tot:6.2f}%   {c / st['attempts']:9.1f} cycles/attempt")
