"""Dump the per-trajectory outputs of configs under the library in $QTM_LIB, or
compare two dumps bit for bit (a refactoring that keeps the arithmetic must
keep every bit: series, jump logs, counters, status).

    QTM_LIB=... python tools/lib_dump.py dump OUT.npz c4:512:39 c5:128:27 c2:4000:-1:lfsr113 ...
    (spec = config[+bdf]:trajectories[:variant[:stream]])
    python tools/lib_dump.py cmp A.npz B.npz
"""
import os, sys
import numpy as np
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def dump(out_path, specs):
    from paper_1810_03047_b200 import configs
    from paper_1810_03047_b200.engine import DeviceProblem, run_logged
    from paper_1810_03047_b200.packing import pack_problem
    arrs = {}
    for spec in specs:
        parts = spec.split(":")
        name, n = parts[0], parts[1]
        v = parts[2] if len(parts) > 2 else "-1"
        stream = parts[3] if len(parts) > 3 else "philox"
        method = None
        if name.endswith("+bdf"):
            name, method = name[:-4], "bdf"
        kw = {}
        if method:
            from paper_1810_03047_b200.problem import OdeConfig
            kw["ode"] = OdeConfig(rtol=1e-8, atol=1e-10, method="bdf")
        pk = pack_problem(configs.build(name, **kw))
        with DeviceProblem(pk, variant=int(v)) as dp:
            out = run_logged(dp, 987654321, 0, int(n), stream=stream)
        key = spec.replace(":", "_").replace("+", "_")
        arrs[key + "_values"] = out.values
        arrs[key + "_stats"] = out.stats
        arrs[key + "_status"] = out.status
        arrs[key + "_jump_count"] = out.jump_count
        arrs[key + "_jump_t"] = out.jump_t
        arrs[key + "_jump_idx"] = out.jump_idx
        arrs[key + "_sum"] = out.sum
        arrs[key + "_sumsq"] = out.sumsq
        print(f"{spec}: kernel {out.kernel_ms:.2f} ms, variant {out.variant}", flush=True)
    np.savez(out_path, **arrs)


def cmp(a_path, b_path):
    a, b = np.load(a_path), np.load(b_path)
    bad = 0
    for k in a.files:
        x, y = a[k], b[k]
        if k.endswith("_jump_t") or k.endswith("_jump_idx"):
            # only the logged part of each row is defined
            cnt = a[k[:k.rindex("_jump_")] + "_jump_count"]
            mask = np.arange(x.shape[1])[None, :] < cnt[:, None]
            x, y = np.where(mask, x, 0), np.where(mask[:, :y.shape[1]], y, 0) if x.shape == y.shape else y
        if x.shape != y.shape:
            print(f"{k}: shape {x.shape} vs {y.shape}"); bad += 1; continue
        same = np.array_equal(x.view(np.uint8) if x.dtype.kind == "f" else x,
                              y.view(np.uint8) if y.dtype.kind == "f" else y)
        if not same:
            bad += 1
            d = np.abs(x.astype(np.float64) - y.astype(np.float64))
            print(f"{k}: DIFFERS, max |d| = {np.nanmax(d):.3e}, {np.count_nonzero(d)} of {d.size} entries")
        else:
            print(f"{k}: bitwise identical")
    print("RESULT:", "identical" if bad == 0 else f"{bad} arrays differ")
    return bad


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(sys.argv[2], sys.argv[3:])
    else:
        sys.exit(1 if cmp(sys.argv[2], sys.argv[3]) else 0)
