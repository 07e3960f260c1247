"""The five BASELINE.json configs, built with this package's constructors.

Concrete inputs follow SURVEY.md §8d (reference basis: index 0 = ground /
spin-up for sigma_z = diag(1, -1)); method ADAMS, rtol 1e-8, atol 1e-10.
tests/test_host_problem.py checks each against the reference-built arrays
stored in tests/golden/<name>.npz.

| name | d    | problem                                   | N       | grid           |
|------|------|-------------------------------------------|---------|----------------|
| c1   | 2    | driven damped two-level atom              | 500     | [0,20], 201 pts|
| c2   | 20   | driven damped cavity                      | 5 000   | [0,30], 301 pts|
| c3   | 80   | Jaynes-Cummings cavity + atom (dense G)   | 20 000  | [0,50], 501 pts|
| c4   | 1024 | dissipative transverse-field Ising, L=10  | 4 096   | [0,10], 101 pts|
| c5   | 900  | two coupled lossy Kerr cavities           | 100 000 | [0,40], 401 pts|
"""

from __future__ import annotations

from math import sqrt

from .csr import dagger, tensor
from .problem import OdeConfig, QuantumProblem, RunOptions
from .qops import (OperatorSet, coherent, destroy, eye, fock, sigma_minus, sigma_x,
                   sigma_z)

__all__ = ["BASELINE_ODE", "CONFIGS", "EXTRA", "N_TRAJECTORIES", "DENSE", "build"]

BASELINE_ODE = OdeConfig(rtol=1e-8, atol=1e-10)
N_TRAJECTORIES = {"c1": 500, "c2": 5_000, "c3": 20_000, "c4": 4_096, "c5": 100_000}
DENSE = {"c3"}  # BASELINE.json marks c3 as the dense-H_eff path


def _mk(ops, psi0, t_to, n_steps, log_jumps, ode):
    return QuantumProblem.from_operators(ops, psi0, 0.0, t_to, n_steps,
                                         ode=ode or BASELINE_ODE,
                                         options=RunOptions(log_jumps=log_jumps))


def c1(log_jumps=False, ode=None):
    """d=2: H = (Omega/2) sigma_x, C = sqrt(0.1) sigma_-, E = [sigma_z, sigma_+ sigma_-]."""
    sm = sigma_minus()
    ops = OperatorSet(0.5 * sigma_x(), (sqrt(0.1) * sm,), (sigma_z(), dagger(sm) @ sm))
    return _mk(ops, fock(2, 0), 20.0, 200, log_jumps, ode)


def c2(log_jumps=False, ode=None):
    """d=20: H = 0.5 a^+a + (a + a^+), C = sqrt(0.5) a, E = [a^+a, (a+a^+)/2]."""
    a = destroy(20)
    ad = dagger(a)
    ops = OperatorSet(0.5 * (ad @ a) + 1.0 * (a + ad), (sqrt(0.5) * a,), (ad @ a, (a + ad) / 2))
    return _mk(ops, coherent(20, 2.0), 30.0, 300, log_jumps, ode)


def c3(log_jumps=False, ode=None):
    """d=80: Jaynes-Cummings, C = [sqrt(0.05) a, sqrt(0.02) sigma_-], E = [a^+a, sigma_z]."""
    a = tensor(destroy(40), eye(2))
    sm = tensor(eye(40), sigma_minus())
    sz = tensor(eye(40), sigma_z())
    ad = dagger(a)
    h = ad @ a + 0.5 * sz + 0.1 * (ad @ sm + a @ dagger(sm))
    ops = OperatorSet(h, (sqrt(0.05) * a, sqrt(0.02) * sm), (ad @ a, sz))
    return _mk(ops, tensor(coherent(40, 3.0), fock(2, 1)), 50.0, 500, log_jumps, ode)


def _site(op, i, n_sites=10):
    factors = [eye(2)] * n_sites
    factors[i] = op
    return tensor(*factors)


def c4(log_jumps=False, ode=None):
    """d=1024: H = -sum sz_i sz_{i+1} - 0.7 sum sx_i (open), C_i = sqrt(0.05) s-_i,
    E_i = sz_i, psi0 = |up...up> = fock(1024, 0)."""
    n_sites = 10
    sz = [_site(sigma_z(), i) for i in range(n_sites)]
    sx = [_site(sigma_x(), i) for i in range(n_sites)]
    h = sum(-1.0 * (sz[i] @ sz[i + 1]) for i in range(n_sites - 1))
    h = h + sum(-0.7 * sx[i] for i in range(n_sites))
    collapse = tuple(sqrt(0.05) * _site(sigma_minus(), i) for i in range(n_sites))
    return _mk(OperatorSet(h, collapse, tuple(sz)), fock(1024, 0), 10.0, 100, log_jumps, ode)


def c5(log_jumps=False, ode=None):
    """d=900: two Kerr cavities, J=1, U=0.2, F=0.5, kappa=0.2, vacuum start."""
    a1 = tensor(destroy(30), eye(30))
    a2 = tensor(eye(30), destroy(30))
    n1 = dagger(a1) @ a1
    n2 = dagger(a2) @ a2
    h = (0.0 * (n1 + n2) + 1.0 * (dagger(a1) @ a2 + dagger(a2) @ a1)
         + 0.2 * (dagger(a1) @ dagger(a1) @ a1 @ a1 + dagger(a2) @ dagger(a2) @ a2 @ a2)
         + 0.5 * (a1 + dagger(a1)))
    ops = OperatorSet(h, (sqrt(0.2) * a1, sqrt(0.2) * a2), (n1, n2))
    return _mk(ops, fock(900, 0), 40.0, 400, log_jumps, ode)


def c4td(log_jumps=False, ode=None):
    """c4 with a modulated transverse field (time-dependent H, timedep.py):
    H(t) = -sum sz_i sz_{i+1} - h(t) sum sx_i, h(t) = 0.7 + 0.3 cos(2 t) --
    the static part in G0, the modulation as one term c(t) = 0.3 cos(2 t)
    on -sum sx_i.  Not a BASELINE config: the measured case of the H(t) row."""
    from .timedep import Coefficient, TimeDependentGenerator
    n_sites = 10
    sz = [_site(sigma_z(), i) for i in range(n_sites)]
    sx = sum(_site(sigma_x(), i) for i in range(n_sites))
    h0 = sum(-1.0 * (sz[i] @ sz[i + 1]) for i in range(n_sites - 1)) - 0.7 * sx
    collapse = tuple(sqrt(0.05) * _site(sigma_minus(), i) for i in range(n_sites))
    gen = TimeDependentGenerator.from_operators(OperatorSet(h0, collapse, ()),
                                                [(-1.0 * sx, Coefficient(0.3, 2.0))])
    from .csr import to_csr
    return QuantumProblem(generator=None, rhs_fn=gen,
                          collapse_csr=tuple(to_csr(c) for c in collapse),
                          expect_csr=tuple(to_csr(z) for z in sz), psi0=fock(1024, 0),
                          t_from=0.0, t_to=10.0, n_steps=100, ode=ode or BASELINE_ODE,
                          options=RunOptions(log_jumps=log_jumps))


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
EXTRA = {"c4td": c4td}
N_TRAJECTORIES["c4td"] = 4_096


def build(name: str, **kw) -> QuantumProblem:
    if name in EXTRA:
        return EXTRA[name](**kw)
    if name not in CONFIGS:
        raise ValueError(f"unknown config {name!r}; expected one of {sorted(CONFIGS)}")
    return CONFIGS[name](**kw)
