"""Generate the BASELINE-scale reference fixtures ``tests/golden/scale_<cN>.npz``.

Run in the build container (needs /root/reference; uses every host core):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_scale_golden.py [c1 c2 ...]

For each BASELINE config this runs the REFERENCE ITSELF
(``mcwf.trajectory.run_single_trajectory``, trajectory.py:190-250) and stores:

* **identical streams** -- every trajectory of c1 (500) and the first 256 of
  c2-c5, once under per-trajectory Philox streams and once under the
  reference's own LFSR113 generator seeded with ``derive_stream(seed, k)``
  (rng.py:76-90): expectation series, jump log (t*, channel), draws consumed,
  the ISTATE of any ``OdeFailure`` (values NaN then) and psi at a few grid
  points for the first ``N_PSI`` trajectories (captured by wrapping the
  module-global ``record_expectation``, trajectory.py:206-214);
* **the reference's own ensemble** -- what ``run_local_farm(problem, N_cpu, K,
  seed)`` computes (cluster.py:493-516): K workers, worker r integrating its
  ``partition_trajectories`` share (cluster.py:369-377) sequentially on ONE
  LFSR113 stream ``derive_stream(seed, r)`` (run_worker, cluster.py:415-420).
  The worker loop is replayed here trajectory by trajectory so the
  per-trajectory values (hence sums of squares, for standard errors) are
  kept; for c1 the mean is checked against a real ``run_local_farm`` call.
  N_cpu follows BASELINE.md's CPU-baseline plan: c1 500, c2 5000, c3 2000,
  c4 4096, c5 256;
* c4 only: the two Philox trajectories of the 4096 ensemble on which the
  reference's Adams controller collapses (``OdeFailure(-5)``), with the
  exception text.

The GPU box only reads these files (tests/test_gpu_scale.py).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

import ref_configs  # noqa: E402  (puts /root/reference/pkg/src on sys.path)
from mcwf import cluster as ref_cluster  # noqa: E402
from mcwf import rng as ref_rng  # noqa: E402
from mcwf import trajectory as ref_traj  # noqa: E402
from mcwf.ode import OdeFailure  # noqa: E402

from oracle.streams import Lfsr113Stream, PhiloxStream  # noqa: E402

SEED = 987654321  # reference DEFAULT_SEED, rng.py:25
N_IDENT = {"c1": 500, "c2": 256, "c3": 256, "c4": 256, "c5": 256}
N_CPU = {"c1": 500, "c2": 5000, "c3": 2000, "c4": 4096, "c5": 256}
K_WORKERS = 8  # run_local_farm worker count of the replayed ensemble
N_PSI = 16
PSI_POINTS = {"c1": [0, 50, 100, 200], "c2": [0, 100, 200, 300], "c3": [0, 125, 250, 500],
              "c4": [0, 25, 50, 100], "c5": [0, 100, 200, 400]}
C4_FAILURES = [3016, 3438]

_PROBLEMS: dict = {}


def _problem(name):
    if name not in _PROBLEMS:
        _PROBLEMS[name] = ref_configs.CONFIGS[name]()
    return _PROBLEMS[name]


class _PsiCapture:
    def __init__(self):
        self.calls = []
        self.orig = ref_traj.record_expectation

    def __enter__(self):
        orig = self.orig

        def wrapped(psi, e):
            self.calls.append(np.array(psi, copy=True))
            return orig(psi, e)
        ref_traj.record_expectation = wrapped
        return self

    def __exit__(self, *exc):
        ref_traj.record_expectation = self.orig


def _one(p, stream, want_psi, psi_points):
    """One reference trajectory; returns (values, jumps, status, msg, psi)."""
    n_e = len(p.expect_csr)
    n_pts = p.n_steps + 1
    psi = None
    try:
        if want_psi:
            with _PsiCapture() as cap:
                res, stream = ref_traj.run_single_trajectory(p, stream)
            per_point = cap.calls[::n_e]
            psi = np.stack([per_point[g] for g in psi_points])
        else:
            res, stream = ref_traj.run_single_trajectory(p, stream)
    except OdeFailure as exc:
        return np.full((n_e, n_pts), np.nan), [], int(exc.istate), str(exc), None, stream
    return res.values, list(res.jumps or []), 0, "", psi, stream


def ident_task(args):
    """Identical-stream chunk: trajectories `ks` under per-trajectory streams."""
    name, kind, ks = args
    p = _problem(name)
    out = []
    for k in ks:
        st = PhiloxStream(SEED, k) if kind == "philox" else Lfsr113Stream(SEED, k)
        vals, jumps, status, msg, psi, st = _one(p, st, k < N_PSI, PSI_POINTS[name])
        out.append((k, vals, jumps, status, msg, psi, st.n if hasattr(st, "n") else -1))
    return out


def farm_task(args):
    """Replay of one run_local_farm worker (cluster.py:415-420)."""
    name, rank, count = args
    p = _problem(name)
    state = ref_rng.derive_stream(SEED, rank)
    vals, jc, fail = [], [], None
    for i in range(count):
        v, jumps, status, msg, _, state2 = _one(p, state, False, [])
        if status:
            # the reference worker would report Error and stop here
            fail = (rank, i, status, msg)
            break
        state = state2
        vals.append(v)
        jc.append(len(jumps))
    return rank, np.asarray(vals), np.asarray(jc, np.int64), fail


def _pack_ident(name, kind, rows, n):
    rows = sorted(rows, key=lambda r: r[0])
    assert [r[0] for r in rows] == list(range(n))
    d = _problem(name).dim
    jt, ji = [], []
    for r in rows:
        jt.extend(t for t, _ in r[2])
        ji.extend(i for _, i in r[2])
    psi = np.stack([r[5] if r[5] is not None else np.zeros((len(PSI_POINTS[name]), d), complex)
                    for r in rows[:N_PSI]])
    return {f"{kind}_traj": np.arange(n, dtype=np.int64),
            f"{kind}_values": np.stack([r[1] for r in rows]),
            f"{kind}_jump_count": np.asarray([len(r[2]) for r in rows], np.int64),
            f"{kind}_jump_t": np.asarray(jt, float), f"{kind}_jump_idx": np.asarray(ji, np.int64),
            f"{kind}_status": np.asarray([r[3] for r in rows], np.int64),
            f"{kind}_n_draws": np.asarray([r[6] for r in rows], np.int64),
            f"{kind}_psi_points": np.asarray(PSI_POINTS[name], np.int64),
            f"{kind}_psi": psi, f"{kind}_n_psi": np.int64(min(N_PSI, n))}


def _farm_mean(p, per_worker):
    """run_master's average: per-worker partials (run_worker), then the
    count-weighted average of the partials (cluster.py:424, 469)."""
    tr = ref_traj.TrajectoryResult
    partials = [ref_traj.average_trajectories([tr(p.time_grid(), v, 1, None) for v in w])
                for w in per_worker if len(w)]
    return ref_traj.average_trajectories(partials).values


def make(name, pool):
    t0 = time.time()
    p = _problem(name)
    n = N_IDENT[name]
    out = {"seed": np.uint64(SEED), "n_ident": np.int64(n)}
    chunks = [list(range(i, n, 16)) for i in range(16)]
    for kind in ("philox", "lfsr113"):
        rows = [r for part in pool.map(ident_task, [(name, kind, c) for c in chunks]) for r in part]
        out.update(_pack_ident(name, kind, rows, n))
        print(f"  {name} {kind}: {time.time() - t0:.0f}s", flush=True)
    counts = ref_cluster.partition_trajectories(N_CPU[name], K_WORKERS)
    parts = sorted(pool.map(farm_task, [(name, r, c) for r, c in enumerate(counts)]),
                   key=lambda x: x[0])
    fails = [f for _, _, _, f in parts if f is not None]
    vals = np.concatenate([v for _, v, _, _ in parts if len(v)])
    out.update(farm_workers=np.int64(K_WORKERS), farm_counts=np.asarray(counts, np.int64),
               farm_n=np.int64(vals.shape[0]), farm_sum=vals.sum(axis=0),
               farm_sumsq=(vals ** 2).sum(axis=0),
               farm_mean=_farm_mean(p, [v for _, v, _, _ in parts]),
               farm_jumps=np.concatenate([j for _, _, j, _ in parts]),
               farm_failures=np.asarray([f[:3] for f in fails], np.int64).reshape(-1, 3))
    print(f"  {name} farm ({N_CPU[name]} on {K_WORKERS} streams, {len(fails)} worker "
          f"failures): {time.time() - t0:.0f}s", flush=True)
    if name == "c1":
        # the replay is run_local_farm itself: same partition, same streams
        real = ref_cluster.run_local_farm(p, N_CPU[name], K_WORKERS, SEED)
        np.testing.assert_allclose(real.values, out["farm_mean"], rtol=0, atol=0)
        out["farm_mean_run_local_farm"] = real.values
    if name == "c4":
        msgs, st = [], []
        for k in C4_FAILURES:
            _, _, status, msg, _, _ = _one(p, PhiloxStream(SEED, k), False, [])
            st.append(status)
            msgs.append(msg)
        out.update(fail_traj=np.asarray(C4_FAILURES, np.int64),
                   fail_status=np.asarray(st, np.int64), fail_msg=np.asarray(msgs))
        print(f"  c4 failures {C4_FAILURES}: {st}", flush=True)
    path = os.path.join(HERE, f"scale_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KB) in {time.time() - t0:.0f}s",
          flush=True)


def main(names):
    for name in names:  # build problems + warm numba in the parent, before the fork
        _problem(name)
    ref_traj.run_single_trajectory(_problem(names[0]), PhiloxStream(SEED, 0))
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        for name in names:
            make(name, pool)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
