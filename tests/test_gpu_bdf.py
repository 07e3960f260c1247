"""BDF on the device (csrc/qtm_bdf.cuh) vs the reference's BDF engine
(golden fixtures from ``mcwf`` with OdeConfig(method="bdf"), ode.py:334-423)
and vs the C oracle's restatement under identical streams.

Same bar as the Adams path: jump sequences exact, series and jump times
within 1e-6.  The LU and the triangular solves have no reductions, so the
device and the oracle differ only through the WRMS/expectation sums (tree
vs sequential) and CUDA's hypot/pow.
"""

import numpy as np
import pytest

import goldens
from paper_1810_03047_b200.engine import DeviceProblem, run_gpu
from paper_1810_03047_b200.packing import pack_problem
from paper_1810_03047_b200.problem import BDF, OdeConfig, QuantumProblem, RunOptions
from paper_1810_03047_b200.qops import OperatorSet, coherent, dagger, destroy

pytestmark = pytest.mark.gpu

TOL = 1e-6
MAXJ = 256


def _compare(out, ref_vals, ref_jc, ref_jt, ref_ji, tol=TOL):
    n = len(ref_jc)
    np.testing.assert_array_equal(out.jump_count[:n], ref_jc)
    for i in range(n):
        m = int(ref_jc[i])
        np.testing.assert_array_equal(out.jump_idx[i, :m], ref_ji[i][:m])
        np.testing.assert_allclose(out.jump_t[i, :m], ref_jt[i][:m], rtol=0, atol=tol)
    np.testing.assert_allclose(out.values[:n], ref_vals, rtol=0, atol=tol)


@pytest.mark.parametrize("name", goldens.BDF_NAMES)
def test_bdf_device_matches_reference_goldens(name):
    g = goldens.load(name)
    assert g.problem.ode.method == BDF
    for kind, s in g.samples.items():
        k0, k1 = int(s.traj[0]), int(s.traj[-1]) + 1
        with DeviceProblem(g.problem) as dp:
            out = dp.run(goldens.SEED, k0, k1, stream=kind, max_jumps=MAXJ, psi_points=s.psi_points,
                         script=goldens.SCRIPTS.get(name))
        assert out.rc == 0, out.error
        _compare(out, s.values, s.jump_count, s.jump_t, s.jump_idx)
        np.testing.assert_array_equal(out.stats[:, 11], s.n_draws)
        if len(s.psi_points):  # psi(t_j) within 1e-6 of the reference's recorded states
            np.testing.assert_allclose(out.psi, s.psi, rtol=0, atol=TOL)


def _cavity(n_fock, kappa=0.5, t_to=10.0, n_steps=100):
    a = destroy(n_fock)
    ad = dagger(a)
    ops = OperatorSet(0.5 * (ad @ a) + 1.0 * (a + ad), (np.sqrt(kappa) * a,), (ad @ a, (a + ad) / 2))
    return QuantumProblem.from_operators(ops, coherent(n_fock, 2.0), 0.0, t_to, n_steps,
                                         ode=OdeConfig(method=BDF, rtol=1e-8, atol=1e-10),
                                         options=RunOptions(log_jumps=True))


# d = 20: workspace in shared memory (32 threads); d = 80, 150: the d^2
# inverse and the vectors in a per-CTA slice of HBM/L2 (128 threads, 4
# trajectories per SM); d = 300: HBM, 256 threads, blocked LU
@pytest.mark.parametrize("name,n", [("bdf_c2", 256), ("bdf_c3", 48), ("cav150", 12), ("cav300", 4)])
def test_bdf_device_matches_oracle(name, n, oracle_lib):
    p = goldens.load(name).problem if name.startswith("bdf_") else \
        _cavity(int(name[3:]), t_to=5.0, n_steps=50)
    pk = pack_problem(p)
    with DeviceProblem(pk) as dp:
        lay = dp.layout()
        out = dp.run(goldens.SEED, 0, n, max_jumps=MAXJ)
    assert out.rc == 0, out.error
    assert (lay["smem_rows"] > 0) == (pk.dim <= 64)
    ref = oracle_lib.run(pk, goldens.SEED, 0, n, max_jumps=MAXJ)
    assert ref["rc"] == 0
    _compare(out, ref["values"], ref["jump_count"],
             [ref["jump_t"][i] for i in range(n)], [ref["jump_idx"][i] for i in range(n)])
    # same step / Newton / rejection counts as the restatement (totals; a
    # rounding-level tie can flip one accept/reject decision in a long run)
    for col in (0, 1, 2, 3, 5):
        a, b = int(out.stats[:, col].sum()), int(ref["stats"][:, col].sum())
        assert abs(a - b) <= max(2, 0.005 * b), (col, a, b)
    np.testing.assert_allclose(out.sum / n, ref["values"].mean(axis=0), rtol=0, atol=TOL)


def test_bdf_shared_memory_workspace_d80(monkeypatch, oracle_lib):
    """c3 BDF with the whole workspace in shared memory (one 256-thread CTA
    per SM, the round-1 placement; forced): same trajectories as the oracle."""
    monkeypatch.setenv("QTM_BDF_HBM", "0")
    monkeypatch.setenv("QTM_BDF_THREADS", "256")
    pk = pack_problem(goldens.load("bdf_c3").problem)
    n = 24
    with DeviceProblem(pk) as dp:
        assert dp.layout()["smem_rows"] > 0
        out = dp.run(goldens.SEED, 0, n, max_jumps=MAXJ)
    assert out.rc == 0, out.error
    ref = oracle_lib.run(pk, goldens.SEED, 0, n, max_jumps=MAXJ)
    _compare(out, ref["values"], ref["jump_count"],
             [ref["jump_t"][i] for i in range(n)], [ref["jump_idx"][i] for i in range(n)])


def test_bdf_run_gpu_end_to_end(oracle_lib):
    g = goldens.load("bdf_stiff")
    res = run_gpu(g.problem, 512, goldens.SEED)
    assert res.n_trajectories == 512
    ref = oracle_lib.run(pack_problem(g.problem), goldens.SEED, 0, 512)
    np.testing.assert_allclose(res.values, ref["values"].mean(axis=0), rtol=0, atol=TOL)
    # the stiff cavity stays near its driven steady state: <a^dag a> bounded
    assert np.all(res.values[0] >= 0.0) and np.all(res.values[0] < 2.0)


def test_bdf_forced_jump_at_ln2():
    g = goldens.load("bdf_decay_forced_jump")
    with DeviceProblem(g.problem) as dp:
        out = dp.run(0, 0, 1, stream="scripted", script=goldens.SCRIPTS["bdf_decay_forced_jump"],
                     max_jumps=4)
    assert out.jump_count[0] == 1 and abs(out.jump_t[0, 0] - np.log(2.0)) < 1e-6


@pytest.mark.parametrize("mode", ["lu", "inv"])
@pytest.mark.parametrize("name,n", [("bdf_c2", 64), ("cav150", 6)])
def test_bdf_solve_modes_agree(mode, name, n, monkeypatch, oracle_lib):
    """Substitution (zgetrs order, bit-identical LU + solve to the oracle)
    and explicit-inverse (zgetri) Newton solves, forced either way."""
    monkeypatch.setenv("QTM_BDF_SOLVE", mode)
    p = goldens.load(name).problem if name.startswith("bdf_") else \
        _cavity(int(name[3:]), t_to=5.0, n_steps=50)
    pk = pack_problem(p)
    with DeviceProblem(pk) as dp:
        out = dp.run(goldens.SEED, 0, n, max_jumps=MAXJ)
    assert out.rc == 0, out.error
    ref = oracle_lib.run(pk, goldens.SEED, 0, n, max_jumps=MAXJ)
    _compare(out, ref["values"], ref["jump_count"],
             [ref["jump_t"][i] for i in range(n)], [ref["jump_idx"][i] for i in range(n)])


def test_bdf_and_adams_agree_at_full_size():
    """c2 at BASELINE size (5 000 trajectories), same Philox streams, both
    method families on the device: two different integrators of the same
    jump process (rtol 1e-8) give the same jump sequences for almost every
    trajectory and ensemble series far inside the statistical error."""
    import dataclasses
    from paper_1810_03047_b200 import configs
    p = configs.build("c2")
    pb = dataclasses.replace(p, ode=OdeConfig(method=BDF, rtol=p.ode.rtol, atol=p.ode.atol))
    n = 5000
    with DeviceProblem(p) as da:
        a = da.run(goldens.SEED, 0, n, max_jumps=MAXJ)
    with DeviceProblem(pb) as db:
        b = db.run(goldens.SEED, 0, n, max_jumps=MAXJ)
    assert a.rc == 0 and b.rc == 0
    same = a.jump_count == b.jump_count
    assert same.mean() > 0.99
    ma, mb = a.sum / n, b.sum / n
    se = np.sqrt(np.maximum(a.sumsq / n - ma ** 2, 0) / n)
    assert np.all(np.abs(ma - mb) <= 2 * se + 1e-6)
    # where the jump sequences agree the series agree to the ODE tolerance
    # level (a grid point between two slightly different jump times aside)
    assert np.quantile(np.abs(a.values[same] - b.values[same]), 0.999) < 1e-4
