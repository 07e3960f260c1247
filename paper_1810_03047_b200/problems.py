"""The reference CLI's named problems (``mcwf.problems``), restated.

``mcwf --problem NAME`` selects one of four builders
(/root/reference/pkg/src/mcwf/problems.py:21-100); the farm protocol checks
that master and workers built the same problem through a 64-bit digest of
its arrays (cluster.py:207-240), so these builders must reproduce the
reference's operators bit for bit -- tests/test_farm.py pins them against
the reference's own digests (tests/golden/farm_wire.json).

    name       dim  physics
    unitary      2  driven qubit, H = (2 pi/10) sigma_x, collapse 0.05 sigma_x
    trilinear  512  three 8-level modes, H = i K (a b+ c+ - a+ b c), damped
    jcm         80  Jaynes-Cummings, 40 levels x qubit, no dissipation
    photon       5  lossy cavity at thermal occupation 0.063
"""

from __future__ import annotations

from math import pi, sqrt

from .csr import dagger, tensor
from .problem import QuantumProblem
from .qops import OperatorSet, coherent, destroy, eye, fock, sigma_minus, sigma_x, sigma_z

__all__ = ["PROBLEM_BUILDERS", "PROBLEM_DEFAULTS", "build_unitary", "build_trilinear",
           "build_jcm", "build_photon"]

# name -> (n_steps, t_to, n_trajectories) defaults (problems.py:21-27)
PROBLEM_DEFAULTS = {
    "unitary": (200, 10.0, 1000),
    "trilinear": (200, 4.0, 1000),
    "jcm": (600, 35.0, 1),
    "photon": (200, 1.0, 1000),
}


def _problem(h, collapse, expect, psi0, n_steps, t_from, t_to, ode, options):
    return QuantumProblem.from_operators(OperatorSet(h, tuple(collapse), tuple(expect)), psi0,
                                         t_from, t_to, n_steps, ode, options)


def build_unitary(*, n_steps=200, t_from=0.0, t_to=10.0, ode=None, options=None,
                  with_collapse=True) -> QuantumProblem:
    """problems.py:30-38: qubit from |0>, sigma_z observed."""
    collapse = [0.05 * sigma_x()] if with_collapse else []
    return _problem((2.0 * pi / 10.0) * sigma_x(), collapse, [sigma_z()], fock(2, 0),
                    n_steps, t_from, t_to, ode, options)


def build_trilinear(*, n_steps=200, t_from=0.0, t_to=4.0, ode=None,
                    options=None) -> QuantumProblem:
    """problems.py:41-60: pump (coherent, |alpha|^2 = 3) and two vacuum
    modes, damping rates 0.1/0.1/0.4, photon numbers observed."""
    levels = 8
    a = destroy(levels)
    one = eye(levels)
    modes = (tensor(a, one, one), tensor(one, a, one), tensor(one, one, a))
    pump, sig, idl = modes
    h = 1j * 1.0 * (pump @ dagger(sig) @ dagger(idl) - dagger(pump) @ sig @ idl)
    rates = (0.1, 0.1, 0.4)
    collapse = [sqrt(2.0 * g) * m for g, m in zip(rates, modes)]
    expect = [dagger(m) @ m for m in modes]
    psi0 = tensor(coherent(levels, sqrt(3.0)), fock(levels, 0), fock(levels, 0))
    return _problem(h, collapse, expect, psi0, n_steps, t_from, t_to, ode, options)


def build_jcm(*, n_steps=600, t_from=0.0, t_to=35.0, ode=None,
              options=None) -> QuantumProblem:
    """problems.py:63-78: detuning -0.1, coupling 1, alpha = 4, qubit
    excited; the spin excitation b+ b is observed; no collapse channels."""
    levels = 40
    a = tensor(destroy(levels), eye(2))
    b = tensor(eye(levels), sigma_minus())
    h = -0.1 * (dagger(a) @ a) + 1.0 * (dagger(a) @ b + a @ dagger(b))
    psi0 = tensor(coherent(levels, 4.0), fock(2, 1))
    return _problem(h, [], [dagger(b) @ b], psi0, n_steps, t_from, t_to, ode, options)


def build_photon(*, n_steps=200, t_from=0.0, t_to=1.0, ode=None,
                 options=None) -> QuantumProblem:
    """problems.py:81-93: H = a+ a on 5 levels, kappa = 1/0.129, bath
    occupation 0.063 (emission and absorption channels), from |1>."""
    a = destroy(5)
    kappa, n_th = 1.0 / 0.129, 0.063
    collapse = [sqrt(kappa * (1.0 + n_th)) * a, sqrt(kappa * n_th) * dagger(a)]
    return _problem(dagger(a) @ a, collapse, [dagger(a) @ a], fock(5, 1), n_steps, t_from,
                    t_to, ode, options)


PROBLEM_BUILDERS = {
    "unitary": build_unitary,
    "trilinear": build_trilinear,
    "jcm": build_jcm,
    "photon": build_photon,
}
