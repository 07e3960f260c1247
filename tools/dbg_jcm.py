import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1810_03047_b200 import cli, native
from paper_1810_03047_b200.engine import DeviceProblem
from paper_1810_03047_b200.packing import pack_problem
from oracle import oracle
import dataclasses
for args in (['--problem','jcm'], ['--problem','jcm','--tol','1e-8'], ['--problem','c3','--t-to','35','--steps','600']):
    p = cli.build_problem(cli.parse_args(args))
    for atol in (None, 1e-10):
        q = p if atol is None else dataclasses.replace(p, ode=dataclasses.replace(p.ode, atol=atol))
        pk = pack_problem(q)
        r = oracle.run(pk, 987654321, 0, 1)
        with DeviceProblem(pk) as dp:
            o = dp.run(987654321, 0, 1)
        d = np.abs(o.values[0] - r['values'][0]).max(axis=0)
        bad = np.nonzero(d > 1e-9)[0]
        print(args, atol, "oracle rc", r['rc'], "dev rc", o.rc, "first bad idx", bad[:3], "t", pk.times[bad[:1]],
              "stats o", r['stats'][0][:12].tolist(), "dev", o.stats[0][:12].tolist(), flush=True)
        if len(bad):
            i = bad[0]
            print("   around", [(float(pk.times[j]), float(r['values'][0][0][j]), float(o.values[0][0][j])) for j in range(max(0, i-2), i+2)])
