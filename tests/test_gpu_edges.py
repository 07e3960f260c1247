"""Edge cases of the device path: empty trajectory ranges, problems without
observables, dimensions that are not a multiple of a warp, and states larger
than every shared-memory staging (d = 4096, CSR from L2, history rows in the
overflow scratch) -- each against the C oracle on identical streams."""

import numpy as np
import pytest

from paper_1810_03047_b200.csr import CsrMatrix
from paper_1810_03047_b200.engine import DeviceProblem, run_gpu
from paper_1810_03047_b200.packing import pack_problem
from paper_1810_03047_b200.problem import OdeConfig, QuantumProblem, RunOptions
from paper_1810_03047_b200.qops import (EffectiveGenerator, OperatorSet, coherent, destroy, fock,
                                        sigma_minus, sigma_x, sigma_z)

pytestmark = pytest.mark.gpu

SEED = 987654321
TOL = 1e-6


def _check(pk, n, oracle_lib, **kw):
    with DeviceProblem(pk, **kw) as dp:
        out = dp.run(SEED, 0, n, max_jumps=64)
    ref = oracle_lib.run(pk, SEED, 0, n, max_jumps=64)
    assert out.rc == ref["rc"] == 0, (out.error, ref["error"])
    np.testing.assert_array_equal(out.jump_count, ref["jump_count"])
    for i in range(n):
        m = int(ref["jump_count"][i])
        np.testing.assert_array_equal(out.jump_idx[i, :m], ref["jump_idx"][i, :m])
        np.testing.assert_allclose(out.jump_t[i, :m], ref["jump_t"][i, :m], rtol=0, atol=TOL)
    np.testing.assert_allclose(out.values, ref["values"], rtol=0, atol=TOL)
    return out


def _cavity(n_fock, expect=True, t_to=5.0, n_steps=50):
    a = destroy(n_fock)
    ad = a.conj().T
    ops = OperatorSet(0.4 * (ad @ a) + 0.8 * (a + ad), (np.sqrt(0.3) * a,),
                      (ad @ a, (a + ad) / 2) if expect else ())
    return QuantumProblem.from_operators(ops, coherent(n_fock, 1.5), 0.0, t_to, n_steps,
                                         ode=OdeConfig(rtol=1e-8, atol=1e-10),
                                         options=RunOptions(log_jumps=True))


def test_empty_trajectory_range():
    pk = pack_problem(_cavity(12))
    with DeviceProblem(pk) as dp:
        out = dp.run(SEED, 7, 7)
    assert out.rc == 0 and out.n_failed == 0
    assert np.all(out.sum == 0.0)


def test_no_observables(oracle_lib):
    p = _cavity(12, expect=False)
    res = run_gpu(p, 64, SEED)
    assert res.values.shape == (0, p.n_steps + 1) and res.n_trajectories == 64
    # the jump process itself still matches the oracle
    _check(pack_problem(p), 64, oracle_lib)


@pytest.mark.parametrize("n_fock", [37, 61, 130])
def test_ragged_dimensions(n_fock, oracle_lib):
    _check(pack_problem(_cavity(n_fock)), 32, oracle_lib)


def test_dimension_4096(oracle_lib):
    """12-site dissipative Ising chain: past every shared-memory staging
    (G read as CSR through L2, two history rows in registers)."""
    import scipy.sparse as sp
    n_sites, dim = 12, 2 ** 12

    def site(op, i):  # sparse kron, site 0 leftmost (linalg.py:111-118)
        return sp.kron(sp.kron(sp.identity(2 ** i), sp.csr_matrix(op)),
                       sp.identity(2 ** (n_sites - 1 - i)), format="csr")

    def csr(m):
        m = sp.csr_matrix(m, dtype=np.complex128)
        m.eliminate_zeros()
        m.sort_indices()
        return CsrMatrix(dim, m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data)
    sz = [site(sigma_z(), i) for i in range(n_sites)]
    h = sum(-1.0 * (sz[i] @ sz[i + 1]) for i in range(n_sites - 1))
    h = h + sum(-0.7 * site(sigma_x(), i) for i in range(n_sites))
    cs = [np.sqrt(0.05) * site(sigma_minus(), i) for i in range(n_sites)]
    g = -1j * h
    for c in cs:
        g = g - 0.5 * (c.conj().T @ c)
    p = QuantumProblem(generator=EffectiveGenerator(csr(g)), collapse_csr=tuple(csr(c) for c in cs),
                       expect_csr=(csr(sz[0]), csr(sz[n_sites // 2])), psi0=fock(dim, 0),
                       t_from=0.0, t_to=4.0, n_steps=20, ode=OdeConfig(rtol=1e-8, atol=1e-10),
                       options=RunOptions(log_jumps=True))
    pk = pack_problem(p)
    assert pk.dim == 4096
    _check(pk, 4, oracle_lib)
