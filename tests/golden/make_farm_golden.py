"""Generate tests/golden/farm_wire.json from the REFERENCE farm codec.

Run in the build container (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_farm_golden.py

Records, as produced by the reference itself:
  * ``mcwf.cluster.problem_digest`` (cluster.py:207-240) of the CLI problems
    (problems.py: unitary, trilinear, jcm, photon -- default arguments and
    the CLI's OdeConfig(rtol=1e-7)) and of the benchmark configs c1..c5
    (tests/golden/ref_configs.py, log_jumps on and off);
  * ``mcwf.cluster.encode_message`` bytes (cluster.py:152-168) of one
    message of every tag, including Results with and without a jump log;
  * the reference's averaged partial for a small unitary run, so the
    decoder and the averaging are pinned on real reference output.

The GPU worker (paper_1810_03047_b200/farm.py) must reproduce the digests
bit for bit, or a reference master rejects it (cluster.py:409-412).
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import ref_configs  # noqa: E402  (puts /root/reference/pkg/src on sys.path)
from mcwf import cluster  # noqa: E402
from mcwf.ode import OdeConfig  # noqa: E402
from mcwf.problems import PROBLEM_BUILDERS  # noqa: E402
from mcwf.trajectory import RunOptions, TrajectoryResult  # noqa: E402


def main():
    out = {"digests": {}, "messages": {}}
    for name, builder in sorted(PROBLEM_BUILDERS.items()):
        p = builder(ode=OdeConfig(rtol=1e-7), options=RunOptions())
        out["digests"][f"cli_{name}"] = str(cluster.problem_digest(p))
        p = builder()
        out["digests"][f"default_{name}"] = str(cluster.problem_digest(p))
    for name in ("c1", "c2", "c3", "c4", "c5"):
        for lj in (False, True):
            p = getattr(ref_configs, name)(log_jumps=lj)
            out["digests"][f"{name}_jumps{int(lj)}"] = str(cluster.problem_digest(p))

    times = np.linspace(0.0, 1.0, 3)
    vals = np.array([[0.25, -1.5, 3.0], [1e-300, np.pi, -0.0]])
    msgs = {
        "hello": cluster.Hello(3),
        "init": cluster.Init(987654321, 0xFEDCBA9876543210, 17),
        "compute": cluster.Compute(),
        "shutdown": cluster.Shutdown(),
        "error": cluster.Error(2, "numeric: trajectory 4 of rank 2: HALT é"),
        "result": cluster.Result(TrajectoryResult(times, vals, 12, None)),
        "result_jumps": cluster.Result(TrajectoryResult(times, vals, 5, [(0.125, 1), (0.5, 0)])),
    }
    for k, m in msgs.items():
        out["messages"][k] = cluster.encode_message(m).hex()

    # a real reference partial: unitary, 3 trajectories on the rank-1 stream
    p = PROBLEM_BUILDERS["unitary"](n_steps=20, t_to=2.0, ode=OdeConfig(rtol=1e-7),
                                    options=dataclasses.replace(RunOptions(), log_jumps=True))
    q1, q2 = cluster.QueueTransport.pair()
    import threading
    th = threading.Thread(target=cluster.run_worker, args=(q2, p, 1))
    th.start()
    q1.send(cluster.Init(11, cluster.problem_digest(p), 3))
    q1.send(cluster.Compute())
    res = q1.recv()
    q1.send(cluster.Shutdown())
    th.join()
    out["messages"]["unitary_partial"] = cluster.encode_message(res).hex()
    with open(os.path.join(HERE, "farm_wire.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
