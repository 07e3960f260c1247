"""Host-side mirror of the reference interface: config builders, Adams
tables, the automatic first step, packing and error mapping."""

import numpy as np
import pytest

import goldens
from paper_1810_03047_b200 import configs, engine
from paper_1810_03047_b200.csr import CsrMatrix, csr_matvec, to_csr
from paper_1810_03047_b200.packing import pack_problem
from paper_1810_03047_b200.problem import (BDF, OdeConfig, OdeFailure, QuantumProblem,
                                           TrajectoryResult, adams_tables, auto_step,
                                           average_trajectories)
from paper_1810_03047_b200.qops import OperatorSet, fock, sigma_minus, sigma_x, sigma_z


def _same_csr(a, b, tol):
    assert a.n == b.n
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.col_ind, b.col_ind)
    np.testing.assert_allclose(a.values, b.values, rtol=0, atol=tol)


@pytest.mark.parametrize("name", goldens.CONFIG_NAMES)
def test_config_builders_match_reference(name):
    g = goldens.load(name)
    p = configs.build(name)
    ref = g.problem
    # identical operators where no matrix exponential is involved; coherent
    # states come from scipy's expm instead of the reference's Pade-13 and
    # agree to rounding
    _same_csr(p.generator.g, ref.generator.g, 1e-14)
    assert len(p.collapse_csr) == len(ref.collapse_csr)
    for a, b in zip(p.collapse_csr, ref.collapse_csr):
        _same_csr(a, b, 1e-15)
    for a, b in zip(p.expect_csr, ref.expect_csr):
        _same_csr(a, b, 1e-15)
    np.testing.assert_allclose(p.psi0, ref.psi0, rtol=0, atol=1e-13)
    assert (p.t_from, p.t_to, p.n_steps) == (ref.t_from, ref.t_to, ref.n_steps)
    assert (p.ode.rtol, p.ode.atol, p.ode.max_order) == (1e-8, 1e-10, 12)
    np.testing.assert_array_equal(p.time_grid(), g.raw["prob_times"])


def test_config_sizes_match_survey():
    want = {"c1": (2, 3), "c2": (20, 57), "c3": (80, 158), "c4": (1024, 11264),
            "c5": (900, 4321)}
    for name, (d, nnz) in want.items():
        p = configs.build(name)
        assert p.dim == d and p.generator.g.nnz == nnz


@pytest.mark.parametrize("name", goldens.CONFIG_NAMES + goldens.SCENARIOS)
def test_auto_step_matches_reference(name):
    g = goldens.load(name)
    p = g.problem
    assert auto_step(p.generator.g, p.psi0, p.ode.rtol, p.ode.atol) == g.h0


def test_adams_tables_known_values():
    l, tau1, tau2, tau3 = adams_tables()
    np.testing.assert_array_equal(l[1, :2], [1.0, 1.0])
    assert tau2[1] == 2.0 and tau3[1] == 12.0
    np.testing.assert_allclose(l[2, :3], [0.5, 1.0, 0.5])
    assert abs(tau2[6] - 70.08) < 0.01
    for q in range(1, 13):
        assert l[q, 1] == 1.0 and np.all(l[q, q + 1:] == 0.0)


def test_csr_matvec_is_sequential_and_unfused():
    rng = np.random.default_rng(7)
    m = rng.standard_normal((9, 9)) + 1j * rng.standard_normal((9, 9))
    m[rng.random((9, 9)) < 0.5] = 0
    c = to_csr(m)
    x = rng.standard_normal(9) + 1j * rng.standard_normal(9)
    y = csr_matvec(c, x)
    for i in range(9):
        sr = si = 0.0
        for j in range(c.row_ptr[i], c.row_ptr[i + 1]):
            a, b = c.values[j].real, c.values[j].imag
            xr, xi = x[c.col_ind[j]].real, x[c.col_ind[j]].imag
            sr = sr + (a * xr - b * xi)
            si = si + (a * xi + b * xr)
        assert y[i] == complex(sr, si)


def test_csr_validation():
    with pytest.raises(ValueError):
        CsrMatrix(2, [0, 2, 2], [1, 0], [1.0, 1.0])  # columns not increasing
    with pytest.raises(ValueError):
        CsrMatrix(2, [0, 1, 2], [0, 2], [1.0, 1.0])  # out of range


def test_problem_validation_mirrors_reference():
    ops = OperatorSet(sigma_x(), (), (sigma_z(),))
    with pytest.raises(ValueError):
        QuantumProblem.from_operators(ops, np.array([1.0, 1.0]), 0.0, 1.0, 10)
    with pytest.raises(ValueError):
        QuantumProblem.from_operators(ops, fock(2, 0), 1.0, 1.0, 10)
    with pytest.raises(ValueError):
        OdeConfig(max_order=13)


def test_pack_selects_method_tables():
    p = QuantumProblem.from_operators(OperatorSet(sigma_x(), (), (sigma_z(),)), fock(2, 0),
                                      0.0, 1.0, 10, ode=OdeConfig(method=BDF))
    pk = pack_problem(p)
    assert pk.method == 1 and pk.max_order == 6
    assert pk.tau2[2] == 4.5 and pk.tau1[2] == 1.0  # BDF2 divisors (Adams2: tau2 = 12)
    assert pk.l_table[2 * 13 + 0] == 2.0 / 3.0  # BDF2 l0 = 2/3 (Adams2: 1/2)
    pa = pack_problem(QuantumProblem.from_operators(
        OperatorSet(sigma_x(), (), (sigma_z(),)), fock(2, 0), 0.0, 1.0, 10))
    assert pa.method == 0 and pa.l_table[2 * 13 + 0] == 0.5
    assert pa.digest != pk.digest


def test_pack_rejects_paths_outside_the_device():
    p2 = QuantumProblem(generator=None, collapse_csr=(), expect_csr=(), psi0=fock(2, 0),
                        t_from=0.0, t_to=1.0, n_steps=10, rhs_fn=lambda t, y: y)
    with pytest.raises(ValueError, match="rhs_fn"):
        pack_problem(p2)


def test_packing_layout():
    p = configs.build("c1")
    pk = pack_problem(p)
    assert pk.psi0.dtype == np.float64 and pk.psi0.shape == (4,)
    assert pk.g.values.shape == (2 * pk.g.nnz,)
    assert pk.times.shape == (201,) and pk.times[-1] == 20.0
    assert pk.l_table.shape == (169,)
    assert pack_problem(configs.build("c1")).digest == pk.digest
    assert pack_problem(configs.build("c2")).digest != pk.digest


def test_partition_rule():
    assert engine.partition_trajectories(10, 3) == [4, 3, 3]
    # shards are whole 256-trajectory reduction blocks (bitwise rank-count
    # invariance, engine.shard_range); the blocks follow the same rule
    assert engine.shard_range(10, 3, 0) == (0, 10) and engine.shard_range(10, 3, 1) == (10, 10)
    assert engine.shard_range(3000, 3, 1) == (1024, 2048)
    assert sum(engine.partition_trajectories(4096, 8)) == 4096
    with pytest.raises(ValueError):
        engine.partition_trajectories(0, 2)


def test_error_messages_mirror_reference(oracle_lib):
    g = goldens.load("c1_max_steps")
    pk = pack_problem(g.problem)
    assert pk.max_steps == 1
    r = oracle_lib.run(pk, goldens.SEED, 0, 1)
    assert r["rc"] == -1
    err = dict(r["error"], max_steps=1)
    with pytest.raises(OdeFailure) as exc:
        engine.raise_for_status(r["rc"], err)
    assert str(exc.value) == str(g.raw["max_steps_msg"])
    assert exc.value.istate == -1


def test_error_mapping_kinds():
    with pytest.raises(OdeFailure, match="ISTATE = -5.*corrector failed"):
        engine.raise_for_status(-6, {"t": 1.0, "h": 0.1})
    with pytest.raises(OdeFailure, match="ISTATE = -4"):
        engine.raise_for_status(-4, {"t": 1.0})
    with pytest.raises(RuntimeError, match="bracket"):
        engine.raise_for_status(-10, {"t": 0.0, "h": 1.0, "aux": (0.1, 0.2, 0.5)})
    with pytest.raises(ValueError, match="support"):
        engine.raise_for_status(-11, {})


def test_average_and_standard_error():
    t = np.linspace(0, 1, 3)
    out = average_trajectories([TrajectoryResult(t, np.full((1, 3), 1.0), 2),
                                TrajectoryResult(t, np.full((1, 3), 2.0), 3)])
    np.testing.assert_allclose(out.values, 1.6)
    r = TrajectoryResult(t, np.full((1, 3), 0.5), 4, sumsq=np.full((1, 3), 2.0))
    np.testing.assert_allclose(r.standard_error(), np.sqrt((0.5 - 0.25) * 4 / 3 / 4))


def test_spmv_value_bytes_follow_the_staging_rule():
    """engine.spmv_value_bytes restates build_sell's rule (csrc/qtm_capi.cu): on
    the wide variants a dominant purely imaginary value (>= half the entries)
    loads nothing, other purely imaginary values (>= a quarter) load 8 bytes,
    everything else 16; the narrow variants load 16 per entry."""
    from paper_1810_03047_b200 import configs
    from paper_1810_03047_b200.engine import smem_model, spmv_value_bytes
    from paper_1810_03047_b200.packing import pack_problem

    c4 = pack_problem(configs.build("c4"))
    c5 = pack_problem(configs.build("c5"))
    wide, narrow = (256, 4, 8), (32, 1, 0)
    # c4: 10 240 off-diagonals are i*h (dominant), 1 024 diagonals stay complex
    assert c4.g.nnz == 11264
    assert spmv_value_bytes(c4, wide) == 16 * 1024
    assert spmv_value_bytes(c4, narrow) == 16 * c4.g.nnz
    assert spmv_value_bytes(c4, None) == 16 * c4.g.nnz
    # c5: no dominant value; 3 422 purely imaginary off-diagonals at 8 bytes, 899 diagonals at 16
    assert spmv_value_bytes(c5, wide) == 8 * 3422 + 16 * 899
    st = {"corr_iters": 10, "attempts": 5}
    assert smem_model(st, c4, wide) < smem_model(st, c4, narrow)
    assert smem_model(st, c4, narrow) == 10 * (36 * c4.g.nnz + 40 * 1024) + 5 * 16 * 1024
