"""Pin the C oracle (oracle/mcwf_oracle.c) against the reference itself.

The fixtures in tests/golden/ were produced by the reference's own
``run_single_trajectory`` (see tests/golden/make_golden.py).  Per-trajectory
streams are identical on both sides, so jump sequences must agree exactly
and the expectation series / jump times to within 1e-6 (BASELINE.json's
parity tolerance; in practice the oracle is bit-exact on the small problems
and within ~1e-7 where the reference's BLAS-ordered dot products differ).
"""

import numpy as np
import pytest

import goldens
from paper_1810_03047_b200.packing import pack_problem

TOL = 1e-6


def _check(name, kind, oracle_lib):
    g = goldens.load(name)
    s = g.samples[kind]
    pk = pack_problem(g.problem)
    k0, k1 = int(s.traj[0]), int(s.traj[-1]) + 1
    assert np.array_equal(s.traj, np.arange(k0, k1))
    r = oracle_lib.run(pk, goldens.SEED, k0, k1, stream=kind, script=goldens.SCRIPTS.get(name),
                       psi_points=s.psi_points)
    assert r["rc"] == 0, r["error"]
    # psi(t_j) itself -- the state the reference hands to record_expectation
    if len(s.psi_points):
        np.testing.assert_allclose(r["psi"], s.psi, rtol=0, atol=TOL)
    np.testing.assert_array_equal(r["jump_count"], s.jump_count)
    for i in range(len(s.traj)):
        n = s.jump_count[i]
        np.testing.assert_array_equal(r["jump_idx"][i, :n], s.jump_idx[i])
        np.testing.assert_allclose(r["jump_t"][i, :n], s.jump_t[i], rtol=0, atol=TOL)
    assert np.abs(r["values"] - s.values).max() <= TOL
    np.testing.assert_array_equal(r["stats"][:, 11], s.n_draws)  # draws consumed
    return r, s


@pytest.mark.parametrize("name", goldens.CONFIG_NAMES)
@pytest.mark.parametrize("kind", ["philox", "lfsr113"])
def test_oracle_matches_reference_configs(name, kind, oracle_lib):
    _check(name, kind, oracle_lib)


@pytest.mark.parametrize("name", goldens.SCENARIOS)
def test_oracle_matches_reference_scenarios(name, oracle_lib):
    g = goldens.load(name)
    for kind in g.samples:
        _check(name, kind, oracle_lib)


def test_oracle_bit_exact_on_small_problems(oracle_lib):
    # d <= 5: no BLAS-ordered reduction differs, the restatement is exact
    for name in ("c1", "decay_streams", "rabi_collapse", "photon", "unitary"):
        g = goldens.load(name)
        for kind, s in g.samples.items():
            r = oracle_lib.run(pack_problem(g.problem), goldens.SEED, int(s.traj[0]),
                               int(s.traj[-1]) + 1, stream=kind)
            np.testing.assert_array_equal(r["values"], s.values)


def test_forced_jump_at_ln2(oracle_lib):
    # reference tests/test_trajectory.py:53-67 with ScriptedDraws [0.5, 0.3, 0.9999999]
    g = goldens.load("decay_forced_jump")
    r = oracle_lib.run(pack_problem(g.problem), 0, 0, 1, stream="scripted",
                       script=goldens.SCRIPTS["decay_forced_jump"])
    assert r["jump_count"][0] == 1 and r["jump_idx"][0, 0] == 0
    assert abs(r["jump_t"][0, 0] - np.log(2.0)) < 1e-6
    times = g.problem.time_grid()
    v = r["values"][0, 0]
    np.testing.assert_allclose(v[times < r["jump_t"][0, 0]], -1.0, atol=1e-9)
    np.testing.assert_allclose(v[times > r["jump_t"][0, 0]], 1.0, atol=1e-9)


def test_oracle_threads_do_not_change_results(oracle_lib):
    g = goldens.load("c2")
    pk = pack_problem(g.problem)
    a = oracle_lib.run(pk, 5, 0, 12, n_threads=1)
    b = oracle_lib.run(pk, 5, 0, 12, n_threads=4)
    np.testing.assert_array_equal(a["values"], b["values"])


# ---- BDF (modified Newton + dense LU, ode.py:334-423) ------------------------
@pytest.mark.parametrize("name", goldens.BDF_NAMES)
def test_oracle_matches_reference_bdf(name, oracle_lib):
    g = goldens.load(name)
    assert g.problem.ode.method == "bdf"
    for kind in g.samples:
        r, s = _check(name, kind, oracle_lib)
        assert r["stats"][:, 5].sum() >= r["stats"][:, 1].sum()  # >= 1 Newton iteration per step


def test_oracle_bdf_forced_jump_at_ln2(oracle_lib):
    g = goldens.load("bdf_decay_forced_jump")
    r = oracle_lib.run(pack_problem(g.problem), 0, 0, 1, stream="scripted",
                       script=goldens.SCRIPTS["bdf_decay_forced_jump"])
    assert r["jump_count"][0] == 1 and abs(r["jump_t"][0, 0] - np.log(2.0)) < 1e-6
    # bit-exact on the scalar decay problem (no BLAS-ordered sums at d = 2 with one nonzero)
    np.testing.assert_array_equal(r["values"], g.samples["scripted"].values)


def test_bdf_tables_match_generating_polynomials():
    from paper_1810_03047_b200.problem import bdf_tables
    l, t1, t2, t3 = bdf_tables()
    # q = 1: backward Euler, l = [1, 1], error constant 2 (ode.py:108-119)
    np.testing.assert_array_equal(l[1, :2], [1.0, 1.0])
    assert t2[1] == 2.0 and t3[1] == 3.0
    # q = 2: P = (x+1)(x+2) = 2 + 3x + x^2 -> l = [2/3, 1, 1/3], H_2 = 3/2
    np.testing.assert_allclose(l[2, :3], [2 / 3, 1.0, 1 / 3], rtol=0, atol=0)
    assert t2[2] == 4.5 and t1[2] == 1.0
    assert np.all(l[7:] == 0.0)


# ---- time-dependent H(t) = H0 + sum_k c_k(t) H_k (rhs_fn, ode.py:334-377) ----
@pytest.mark.parametrize("name", goldens.TD_NAMES)
def test_oracle_matches_reference_time_dependent(name, oracle_lib):
    g = goldens.load(name)
    assert g.problem.generator is None and g.problem.rhs_fn is not None
    assert pack_problem(g.problem).h0_first == g.h0  # auto step from G(t_from) psi0
    for kind in g.samples:
        _check(name, kind, oracle_lib)


def test_time_dependent_generator_call_order():
    """The rhs_fn callable adds c_k(t) (G_k psi) to G0 psi term by term --
    the order the oracle and the device kernel use."""
    from paper_1810_03047_b200.csr import csr_matvec
    g = goldens.load("td_cavity")
    gen = g.problem.rhs_fn
    psi = g.problem.psi0 * (1 + 0.5j)
    t = 1.234
    want = csr_matvec(gen.g0, psi)
    for m, c in gen.terms:
        want = want + (c.offset + c.amp * np.cos(c.omega * t + c.phase)) * csr_matvec(m, psi)
    np.testing.assert_array_equal(gen(t, psi), want)
    with pytest.raises(ValueError, match="ADAMS"):
        import dataclasses
        from paper_1810_03047_b200.problem import OdeConfig
        pack_problem(dataclasses.replace(g.problem, ode=OdeConfig(method="bdf")))


# ---- ensemble limit: the unravelling converges to the Lindblad solution ------
@pytest.mark.parametrize("name,n", [("c1", 4000), ("c2", 600)])
def test_oracle_ensemble_converges_to_lindblad(name, n, oracle_lib):
    """The trajectory average vs the reference's dense master-equation
    oracle (solve_master_equation, trajectory.py:276-299; fixture
    tests/golden/lindblad_<name>.npz): within 4.5 standard errors at every
    point, plus the ODE tolerance."""
    import os
    from paper_1810_03047_b200 import configs
    z = np.load(os.path.join(goldens.GOLDEN_DIR, f"lindblad_{name}.npz"))
    r = oracle_lib.run(pack_problem(configs.build(name)), 2024, 0, n)
    mean = r["values"].mean(axis=0)
    se = r["values"].std(axis=0, ddof=1) / np.sqrt(n)
    np.testing.assert_allclose(z["times"], configs.build(name).time_grid(), rtol=0, atol=1e-12)
    # (+1e-3: before the first jumps of a finite ensemble its sample SE is 0
    # while the Lindblad curve already carries the O(t) jump probability)
    assert np.all(np.abs(mean - z["values"]) <= 4.5 * se + 1e-3)
