"""Edge cases of the device path: empty trajectory ranges, problems without
observables, dimensions that are not a multiple of a warp, and states larger
than every shared-memory staging (d = 4096, CSR from L2, history rows in the
overflow scratch) -- each against the C oracle on identical streams."""

import numpy as np
import pytest

from paper_1810_03047_b200.csr import tensor
from paper_1810_03047_b200.engine import DeviceProblem, run_gpu
from paper_1810_03047_b200.packing import pack_problem
from paper_1810_03047_b200.problem import OdeConfig, QuantumProblem, RunOptions
from paper_1810_03047_b200.qops import (OperatorSet, coherent, destroy, eye, fock, sigma_minus,
                                        sigma_x, sigma_z)

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
    n_sites = 12

    def site(op, i):
        f = [eye(2)] * n_sites
        f[i] = op
        return tensor(*f)
    sz = [site(sigma_z(), i) for i in range(n_sites)]
    h = sum(-1.0 * (sz[i] @ sz[i + 1]) for i in range(n_sites - 1))
    h = h + sum(-0.7 * site(sigma_x(), i) for i in range(n_sites))
    ops = OperatorSet(h, tuple(np.sqrt(0.05) * site(sigma_minus(), i) for i in range(n_sites)),
                      (sz[0], sz[n_sites // 2]))
    p = QuantumProblem.from_operators(ops, fock(2 ** n_sites, 0), 0.0, 1.0, 10,
                                      ode=OdeConfig(rtol=1e-8, atol=1e-10),
                                      options=RunOptions(log_jumps=True))
    pk = pack_problem(p)
    assert pk.dim == 4096
    _check(pk, 4, oracle_lib)
