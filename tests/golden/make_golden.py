"""Generate the golden fixtures under tests/golden/ from the REFERENCE.

Run in the build container (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Each ``<name>.npz`` holds
  * the problem exactly as the reference built it (CSR arrays of G, the
    collapse and expectation operators, psi0, grid, ODE config and the
    reference's own automatic first step ``h0``, read back from
    ``OdeSolver.h``, ode.py:199-203, 247-252);
  * per-trajectory outputs of ``mcwf.trajectory.run_single_trajectory``
    (trajectory.py:190-250) under per-trajectory streams from
    ``oracle/streams.py`` (philox / lfsr113 / scripted): the expectation
    series, the jump log (t*, channel), the number of draws consumed and
    snapshots of psi at selected grid points (captured by wrapping the
    module-global ``record_expectation``, which ``record`` looks up at call
    time, trajectory.py:206-214).

The fixtures pin the C oracle (tests/test_oracle_golden.py) and the device
kernels (tests/test_gpu_parity.py).  Nothing on the GPU box reads
/root/reference; it only reads these files.
"""

from __future__ import annotations

import dataclasses
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

import ref_configs  # noqa: E402  (puts /root/reference/pkg/src on sys.path)
import mcwf  # noqa: E402
from mcwf import rng as ref_rng  # noqa: E402
from mcwf import trajectory as ref_traj  # noqa: E402
from mcwf.linalg import to_csr  # noqa: E402
from mcwf.ode import OdeConfig, OdeFailure, OdeSolver  # noqa: E402
from mcwf.operators import OperatorSet, fock, sigma_minus, sigma_x, sigma_z  # noqa: E402
from mcwf.problems import build_photon, build_trilinear, build_unitary  # noqa: E402
from mcwf.trajectory import QuantumProblem, RunOptions  # noqa: E402

from oracle.streams import (Lfsr113Stream, PhiloxStream, ScriptedStream,  # noqa: E402
                            lfsr113_derive)

SEED = 987654321  # reference DEFAULT_SEED, rng.py:25


def problem_arrays(p: QuantumProblem) -> dict:
    out = {"dim": p.dim, "t_from": p.t_from, "t_to": p.t_to, "n_steps": p.n_steps,
           "rtol": p.ode.rtol, "atol": p.ode.atol, "max_order": p.ode.max_order,
           "max_steps": p.ode.max_steps,
           "initial_step": np.nan if p.ode.initial_step is None else p.ode.initial_step,
           "psi0": p.psi0, "times": p.time_grid(),
           "n_collapse": len(p.collapse_csr), "n_expect": len(p.expect_csr)}
    if p.ode.method != "adams":
        out["method"] = p.ode.method
    if p.generator is None:  # TimeDependentGenerator rhs_fn (paper_1810_03047_b200/timedep.py)
        gen = p.rhs_fn
        g = gen.g0
        out["n_td"] = len(gen.terms)
        out["td_coef"] = np.concatenate([c.as_array() for _, c in gen.terms])
        for k, (m, _) in enumerate(gen.terms):
            out[f"td{k}_row_ptr"] = m.row_ptr
            out[f"td{k}_col_ind"] = m.col_ind
            out[f"td{k}_values"] = m.values
    else:
        g = p.generator.g
    out.update(g_row_ptr=g.row_ptr, g_col_ind=g.col_ind, g_values=g.values)
    for tag, ops in (("c", p.collapse_csr), ("e", p.expect_csr)):
        for i, m in enumerate(ops):
            out[f"{tag}{i}_row_ptr"] = m.row_ptr
            out[f"{tag}{i}_col_ind"] = m.col_ind
            out[f"{tag}{i}_values"] = m.values
    out["h0"] = OdeSolver(p.ode, g if p.generator is not None else p.rhs_fn,
                          t0=p.t_from, y0=p.psi0.copy()).h
    return out


class _PsiCapture:
    def __init__(self, dim, n_pts, keep):
        self.keep = set(int(g) for g in keep)
        self.buf = {}
        self.gi = None
        self.orig = ref_traj.record_expectation

    def __enter__(self):
        cap = self
        orig = self.orig

        def wrapped(psi, e):
            cap.calls.append(np.array(psi, copy=True))
            return orig(psi, e)

        self.calls = []
        ref_traj.record_expectation = wrapped
        return self

    def __exit__(self, *exc):
        ref_traj.record_expectation = self.orig


def run_sample(p, kind, indices, psi_points, n_expect, script=None):
    n_pts = p.n_steps + 1
    vals, jcount, jt, jidx, ndraws, psis = [], [], [], [], [], []
    for k in indices:
        if kind == "philox":
            st = PhiloxStream(SEED, k)
        elif kind == "lfsr113":
            st = Lfsr113Stream(SEED, k)
        else:
            st = ScriptedStream(script[k], 0.999999)
        cap = _PsiCapture(p.dim, n_pts, psi_points)
        with cap:
            res, st2 = ref_traj.run_single_trajectory(p, st)
        # record() calls record_expectation once per expectation operator per
        # grid point, in grid order
        per_point = cap.calls[::n_expect]
        assert len(per_point) == n_pts
        psis.append(np.stack([per_point[g] for g in psi_points]) if len(psi_points) else
                    np.zeros((0, p.dim), complex))
        vals.append(res.values)
        jumps = res.jumps or []
        jcount.append(len(jumps))
        jt.extend(t for t, _ in jumps)
        jidx.extend(i for _, i in jumps)
        ndraws.append(st.n if hasattr(st, "n") else 1 + 2 * len(jumps))
    return {"kind": kind, "traj": np.asarray(indices, np.int64),
            "values": np.stack(vals), "jump_count": np.asarray(jcount, np.int64),
            "jump_t": np.asarray(jt, float), "jump_idx": np.asarray(jidx, np.int64),
            "n_draws": np.asarray(ndraws, np.int64),
            "psi_points": np.asarray(psi_points, np.int64), "psi": np.stack(psis)}


def save(name, p, samples, extra=None):
    arrs = {f"prob_{k}": np.asarray(v) for k, v in problem_arrays(p).items()}
    arrs["seed"] = np.uint64(SEED)
    for s in samples:
        tag = s["kind"]
        for k, v in s.items():
            if k != "kind":
                arrs[f"{tag}_{k}"] = np.asarray(v)
    arrs["kinds"] = np.array([s["kind"] for s in samples])
    if extra:
        arrs.update(extra)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrs)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KB)")


def with_log(p):
    return dataclasses.replace(p, options=RunOptions(log_jumps=True))


def main():
    t0 = time.time()
    plan = {  # name: (philox indices, lfsr indices, psi grid points)
        "c1": (list(range(64)), list(range(16)), list(range(0, 201, 5))),
        "c2": (list(range(12)), list(range(4)), list(range(0, 301, 10))),
        "c3": (list(range(6)), list(range(2)), list(range(0, 501, 25))),
        "c4": (list(range(4)), [0], list(range(0, 101, 20))),
        "c5": ([0, 1], [0], list(range(0, 401, 80))),
    }
    for name, (ph, lf, pts) in plan.items():
        p = ref_configs.CONFIGS[name]()
        n_e = len(p.expect_csr)
        samples = [run_sample(p, "philox", ph, pts, n_e),
                   run_sample(p, "lfsr113", lf, pts[:4], n_e)]
        save(name, p, samples)
        print(f"  {name}: {time.time() - t0:.1f}s")

    # reference unit-test scenarios (tests/test_trajectory.py) ----------------
    decay = lambda t_to, n_steps, rtol=1e-8: QuantumProblem.from_operators(  # noqa: E731
        OperatorSet(np.zeros((2, 2), complex), (sigma_minus(),), (sigma_z(),)),
        fock(2, 1), 0.0, t_to, n_steps, ode=OdeConfig(rtol=rtol, atol=1e-12),
        options=RunOptions(log_jumps=True))
    p = decay(12.0, 12)
    scripts = {0: [0.5, 0.3, 0.9999999]}
    save("decay_forced_jump", p, [run_sample(p, "scripted", [0], range(13), 1, scripts)])
    p = decay(1.0, 10)
    scripts = {0: [np.exp(-1.0) / 2]}
    save("decay_no_jump", p, [run_sample(p, "scripted", [0], range(11), 1, scripts)])
    p = decay(12.0, 12)
    save("decay_streams", p, [run_sample(p, "philox", list(range(32)), [], 1),
                              run_sample(p, "lfsr113", list(range(16)), [], 1)])

    omega = 2 * np.pi / 10
    rabi = QuantumProblem.from_operators(
        OperatorSet(omega * sigma_x(), (), (sigma_z(),)), fock(2, 0), 0.0, 10.0, 100,
        ode=OdeConfig(rtol=1e-8, atol=1e-12), options=RunOptions(log_jumps=True))
    save("rabi_closed", rabi, [run_sample(rabi, "philox", [0], list(range(101)), 1)])
    rabi_c = QuantumProblem.from_operators(
        OperatorSet(omega * sigma_x(), (0.05 * sigma_x(),), (sigma_z(),)), fock(2, 0),
        0.0, 10.0, 100, ode=OdeConfig(rtol=1e-8, atol=1e-12),
        options=RunOptions(log_jumps=True))
    save("rabi_collapse", rabi_c, [run_sample(rabi_c, "philox", list(range(32)), [], 1)])

    for name, builder, nph in (("photon", build_photon, 48), ("unitary", build_unitary, 32),
                               ("trilinear", build_trilinear, 2)):
        p = with_log(builder())
        save(name, p, [run_sample(p, "philox", list(range(nph)), [0, p.n_steps // 2],
                                  len(p.expect_csr))])

    # failure scenarios: the exact exception text the boundary must mirror
    msgs = {}
    p = dataclasses.replace(ref_configs.c1(), ode=OdeConfig(rtol=1e-8, atol=1e-10, max_steps=1))
    try:
        ref_traj.run_single_trajectory(p, PhiloxStream(SEED, 0))
    except OdeFailure as exc:
        msgs["max_steps_msg"] = np.array(str(exc))
        msgs["max_steps_istate"] = np.int64(exc.istate)
    save("c1_max_steps", p, [], msgs)

    # LFSR113 stream bits: derive_stream(seed, k) words and first 64 draws
    words, draws = [], []
    for k in range(8):
        st = ref_rng.derive_stream(SEED, k)
        words.append((st.z1, st.z2, st.z3, st.z4))
        assert tuple(lfsr113_derive(SEED, k)) == words[-1]
        row = []
        for _ in range(64):
            u, st = st.next_u01()
            row.append(u)
        draws.append(row)
    np.savez_compressed(os.path.join(HERE, "lfsr113_streams.npz"),
                        seed=np.uint64(SEED), words=np.asarray(words, np.uint64),
                        draws=np.asarray(draws))
    print(f"done in {time.time() - t0:.1f}s  (mcwf {mcwf.__version__})")


def as_bdf(p, **kw):
    ode = OdeConfig(method="bdf", rtol=p.ode.rtol, atol=p.ode.atol, **kw)
    return dataclasses.replace(p, ode=ode)


def main_bdf():
    """BDF fixtures (``bdf_*.npz``): the reference's general engine with the
    modified-Newton corrector and scipy's LU (ode.py:334-437) on the same
    CSR problems, plus a stiff cavity (decay rate >> drive) where BDF is the
    method of choice."""
    t0 = time.time()
    plan = {"c1": (list(range(64)), list(range(16)), list(range(0, 201, 5))),
            "c2": (list(range(16)), list(range(4)), list(range(0, 301, 10))),
            "c3": (list(range(6)), [0], list(range(0, 501, 50)))}
    for name, (ph, lf, pts) in plan.items():
        p = as_bdf(ref_configs.CONFIGS[name]())
        n_e = len(p.expect_csr)
        save(f"bdf_{name}", p, [run_sample(p, "philox", ph, pts, n_e),
                                run_sample(p, "lfsr113", lf, pts[:4], n_e)])
        print(f"  bdf_{name}: {time.time() - t0:.1f}s")
    p = as_bdf(ref_configs.stiff_cavity())
    save("bdf_stiff", p, [run_sample(p, "philox", list(range(64)), list(range(0, 101, 10)),
                                     len(p.expect_csr))])
    print(f"  bdf_stiff: {time.time() - t0:.1f}s")
    decay = QuantumProblem.from_operators(
        OperatorSet(np.zeros((2, 2), complex), (sigma_minus(),), (sigma_z(),)),
        fock(2, 1), 0.0, 12.0, 12, ode=OdeConfig(method="bdf", rtol=1e-8, atol=1e-12),
        options=RunOptions(log_jumps=True))
    save("bdf_decay_forced_jump", decay,
         [run_sample(decay, "scripted", [0], range(13), 1, {0: [0.5, 0.3, 0.9999999]})])
    print(f"bdf fixtures done in {time.time() - t0:.1f}s")


def main_td():
    """Time-dependent fixtures (``td_*.npz``): the reference's general Adams
    engine (ode.py:334-377) driving a ``TimeDependentGenerator`` rhs_fn --
    H(t) = H0 + sum_k c_k(t) H_k -- through ``run_single_trajectory``."""
    from math import sqrt

    from paper_1810_03047_b200 import timedep as ours_td
    from paper_1810_03047_b200 import qops as ours_ops
    from mcwf.linalg import dagger, tensor
    from mcwf.operators import destroy, eye

    t0 = time.time()
    ode = OdeConfig(rtol=1e-8, atol=1e-10)

    def td_problem(h0, h_terms, collapse, expect, psi0, t_to, n_steps):
        gen = ours_td.TimeDependentGenerator.from_operators(
            ours_ops.OperatorSet(h0, tuple(collapse), ()), h_terms)
        return QuantumProblem(generator=None, rhs_fn=gen,
                              collapse_csr=tuple(to_csr(c) for c in collapse),
                              expect_csr=tuple(to_csr(e) for e in expect), psi0=psi0,
                              t_from=0.0, t_to=t_to, n_steps=n_steps, ode=ode,
                              options=RunOptions(log_jumps=True))

    sm = sigma_minus()
    rabi = td_problem(0.5 * sigma_z(), [(sigma_x(), ours_td.Coefficient(0.5, 1.0))],
                      [sqrt(0.1) * sm], [sigma_z(), dagger(sm) @ sm], fock(2, 0), 20.0, 200)
    save("td_rabi", rabi, [run_sample(rabi, "philox", list(range(64)), list(range(0, 201, 10)), 2),
                           run_sample(rabi, "lfsr113", list(range(16)), [], 2)])
    print(f"  td_rabi: {time.time() - t0:.1f}s")
    a = destroy(20)
    ad = dagger(a)
    cav = td_problem(0.5 * (ad @ a), [(a + ad, ours_td.Coefficient(1.0, 0.5)),
                                      (ad @ a, ours_td.Coefficient(0.2, 2.0, 0.3, 0.05))],
                     [sqrt(0.5) * a], [ad @ a, (a + ad) / 2], fock(20, 0), 30.0, 300)
    save("td_cavity", cav, [run_sample(cav, "philox", list(range(12)), list(range(0, 301, 30)), 2)])
    print(f"  td_cavity: {time.time() - t0:.1f}s")
    n_sites = 6

    def site(op, i):
        f = [eye(2)] * n_sites
        f[i] = op
        return tensor(*f)
    sz = [site(sigma_z(), i) for i in range(n_sites)]
    sx = sum(site(sigma_x(), i) for i in range(n_sites))
    h0 = sum(-1.0 * (sz[i] @ sz[i + 1]) for i in range(n_sites - 1)) - 0.7 * sx
    ising = td_problem(h0, [(-1.0 * sx, ours_td.Coefficient(0.3, 2.0))],
                       [sqrt(0.05) * site(sm, i) for i in range(n_sites)], sz,
                       fock(2 ** n_sites, 0), 10.0, 100)
    save("td_ising", ising, [run_sample(ising, "philox", list(range(6)), list(range(0, 101, 20)), 6)])
    print(f"td fixtures done in {time.time() - t0:.1f}s")


def main_lindblad():
    """Ensemble limits (``lindblad_*.npz``): the reference's dense Lindblad
    oracle ``solve_master_equation`` (trajectory.py:276-299) on c1 and c2 --
    what the trajectory average converges to as N grows."""
    from mcwf.trajectory import solve_master_equation
    t0 = time.time()
    for name, build in (("c1", ref_configs.c1_ops), ("c2", ref_configs.c2_ops)):
        ops, psi0, times = build()
        rho0 = np.outer(psi0, psi0.conj())
        vals = solve_master_equation(ops, rho0, times, ode=OdeConfig(rtol=1e-8, atol=1e-10))
        np.savez_compressed(os.path.join(HERE, f"lindblad_{name}.npz"), times=times, values=vals)
        print(f"  lindblad_{name}: {time.time() - t0:.1f}s")


if __name__ == "__main__":
    if "--lindblad" in sys.argv:
        main_lindblad()
    elif "--td" in sys.argv:
        main_td()
    elif "--bdf" in sys.argv:
        main_bdf()
    else:
        main()
