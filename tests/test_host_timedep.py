"""Host side of the time-dependent path (timedep.py) and the BDF packing:
validation, the device form in the packed problem, and the oracle's psi
snapshot output (CPU only)."""

import numpy as np
import pytest

from paper_1810_03047_b200.csr import to_csr
from paper_1810_03047_b200.packing import pack_problem
from paper_1810_03047_b200.problem import OdeConfig, QuantumProblem
from paper_1810_03047_b200.qops import OperatorSet, fock, sigma_minus, sigma_x, sigma_z
from paper_1810_03047_b200.timedep import MAX_TD_TERMS, Coefficient, TimeDependentGenerator


def _gen(n_terms=1):
    ops = OperatorSet(0.5 * sigma_z(), (np.sqrt(0.1) * sigma_minus(),), ())
    return TimeDependentGenerator.from_operators(
        ops, [(sigma_x(), Coefficient(0.5, 1.0 + k)) for k in range(n_terms)])


def _problem(rhs, **kw):
    return QuantumProblem(generator=None, rhs_fn=rhs, collapse_csr=(to_csr(np.sqrt(0.1) * sigma_minus()),),
                          expect_csr=(to_csr(sigma_z()),), psi0=fock(2, 0), t_from=0.0, t_to=1.0,
                          n_steps=10, **kw)


def test_coefficient_form():
    c = Coefficient(2.0, 3.0, 0.25, -1.0)
    assert c(0.5) == -1.0 + 2.0 * np.cos(3.0 * 0.5 + 0.25)
    np.testing.assert_array_equal(c.as_array(), [2.0, 3.0, 0.25, -1.0])


def test_generator_validation():
    with pytest.raises(ValueError):
        TimeDependentGenerator(_gen().g0, [])
    with pytest.raises(ValueError):
        _gen(MAX_TD_TERMS + 1)
    with pytest.raises(ValueError):
        TimeDependentGenerator(_gen().g0, [(to_csr(np.eye(3)), Coefficient(1.0))])


def test_packed_device_form():
    gen = _gen(2)
    pk = pack_problem(_problem(gen))
    assert pk.n_td == 2 and pk.td_coef.shape == (8,)
    np.testing.assert_array_equal(pk.td_coef[:4], [0.5, 1.0, 0.0, 0.0])
    # the first step uses G(t_from) psi0, as the reference's _auto_step(y0, f0)
    f0 = gen(0.0, fock(2, 0))
    w2 = 1.0 / (1e-12 + 1e-7 * np.abs(fock(2, 0))) ** 2
    fw = np.sqrt(float((f0.real * f0.real + f0.imag * f0.imag) @ w2) / 2)
    assert pk.h0_first == 0.01 / fw
    assert pack_problem(_problem(_gen(1))).digest != pk.digest


def test_arbitrary_callbacks_and_bdf_rejected():
    with pytest.raises(ValueError, match="TimeDependentGenerator"):
        pack_problem(_problem(lambda t, y: y))
    with pytest.raises(ValueError, match="ADAMS"):
        pack_problem(_problem(_gen(), ode=OdeConfig(method="bdf")))


def test_oracle_psi_snapshots(oracle_lib):
    pk = pack_problem(_problem(_gen()))
    r = oracle_lib.run(pk, 7, 0, 3, psi_points=[0, 5, 10])
    assert r["psi"].shape == (3, 3, 2)
    np.testing.assert_array_equal(r["psi"][:, 0], np.tile(fock(2, 0), (3, 1)))  # record(0) = psi0
    # the recorded (unnormalised) state reproduces the recorded expectation
    psi = r["psi"][:, 1]
    sz = (np.abs(psi[:, 0]) ** 2 - np.abs(psi[:, 1]) ** 2) / (np.abs(psi) ** 2).sum(axis=1)
    np.testing.assert_allclose(sz, r["values"][:, 0, 5], rtol=0, atol=1e-14)
