import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1810_03047_b200 import configs, native
from paper_1810_03047_b200.problems import PROBLEM_BUILDERS
from paper_1810_03047_b200.engine import DeviceProblem
from paper_1810_03047_b200.packing import pack_problem
from oracle import oracle
for name, p in (("photon", PROBLEM_BUILDERS["photon"]()), ("c1", configs.build("c1")), ("c4", configs.build("c4"))):
    pk = pack_problem(p)
    r = oracle.run(pk, 987654321, 0, 4)
    with DeviceProblem(pk) as dp:
        o = dp.run(987654321, 0, 4)
        o2 = dp.run(987654321, 0, 4, resident=True, per_trajectory=False)
    print(name, native.variants()[o.variant], "rc", o.rc, "dev v0", o.values[0, :, :3].tolist(), "oracle", r["values"][0, :, :3].tolist())
    print("   sum/n dev", (o2.sum / 4)[:, :3].tolist(), "oracle", r["values"].mean(axis=0)[:, :3].tolist())
