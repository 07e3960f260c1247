"""BASELINE configs c1-c5 built with the REFERENCE constructors.

Used by ``make_golden.py`` / ``make_scale_golden.py`` in the build
container (where /root/reference is mounted) and by the drop-in tests
(tests/test_dropin*.py), which import the reference from baseline/_ref when
/root/reference is absent.  The concrete inputs follow SURVEY.md §8d.
"""

from __future__ import annotations

import sys
from math import sqrt

import os

# the reference package: its source tree in the build container, else the
# copy pip-installed into baseline/_ref (travels to the GPU box)
_REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_SRC = next((p for p in ("/root/reference/pkg/src", os.path.join(_REPO, "baseline", "_ref"))
                if os.path.isdir(os.path.join(p, "mcwf"))), None)
if REF_SRC is None:
    raise ImportError("the reference package mcwf is not available (no /root/reference, "
                      "no baseline/_ref)")
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

from mcwf.linalg import dagger, tensor  # noqa: E402
from mcwf.ode import OdeConfig  # noqa: E402
from mcwf.operators import (OperatorSet, coherent, destroy, eye, fock,  # noqa: E402
                            sigma_minus, sigma_x, sigma_z)
from mcwf.trajectory import QuantumProblem, RunOptions  # noqa: E402

# BASELINE.json: rtol=1e-8, atol=1e-10 (stated for c1, applied to all five;
# SURVEY.md §8d records the choice), reference default method ADAMS.
ODE = OdeConfig(rtol=1e-8, atol=1e-10)


def _problem(ops, psi0, t_to, n_steps, log_jumps):
    return QuantumProblem.from_operators(ops, psi0, 0.0, t_to, n_steps, ode=ODE,
                                         options=RunOptions(log_jumps=log_jumps))


def c1_ops():
    sm = sigma_minus()
    ops = OperatorSet(0.5 * sigma_x(), (sqrt(0.1) * sm,), (sigma_z(), dagger(sm) @ sm))
    return ops, fock(2, 0), __import__("numpy").linspace(0.0, 20.0, 201)


def c1(log_jumps=True):
    ops, psi0, _ = c1_ops()
    return _problem(ops, psi0, 20.0, 200, log_jumps)


def c2_ops():
    a = destroy(20)
    ad = dagger(a)
    ops = OperatorSet(0.5 * (ad @ a) + 1.0 * (a + ad), (sqrt(0.5) * a,),
                      (ad @ a, (a + ad) / 2))
    return ops, coherent(20, 2.0), __import__("numpy").linspace(0.0, 30.0, 301)


def c2(log_jumps=True):
    ops, psi0, _ = c2_ops()
    return _problem(ops, psi0, 30.0, 300, log_jumps)


def c3(log_jumps=True):
    a = tensor(destroy(40), eye(2))
    sm = tensor(eye(40), sigma_minus())
    sz = tensor(eye(40), sigma_z())
    ad = dagger(a)
    h = ad @ a + 0.5 * sz + 0.1 * (ad @ sm + a @ dagger(sm))
    ops = OperatorSet(h, (sqrt(0.05) * a, sqrt(0.02) * sm), (ad @ a, sz))
    return _problem(ops, tensor(coherent(40, 3.0), fock(2, 1)), 50.0, 500, log_jumps)


def _site(op, i, n_sites=10):
    factors = [eye(2)] * n_sites
    factors[i] = op
    return tensor(*factors)


def c4(log_jumps=True):
    n_sites = 10
    sz = [_site(sigma_z(), i) for i in range(n_sites)]
    sx = [_site(sigma_x(), i) for i in range(n_sites)]
    h = sum(-1.0 * (sz[i] @ sz[i + 1]) for i in range(n_sites - 1))
    h = h + sum(-0.7 * sx[i] for i in range(n_sites))
    collapse = tuple(sqrt(0.05) * _site(sigma_minus(), i) for i in range(n_sites))
    ops = OperatorSet(h, collapse, tuple(sz))
    # psi0 = |up...up> = fock(1024, 0) under the reference basis (index 0 =
    # sigma_z eigenvalue +1); SURVEY.md §8d records the choice.
    return _problem(ops, fock(1024, 0), 10.0, 100, log_jumps)


def c5(log_jumps=True):
    a1 = tensor(destroy(30), eye(30))
    a2 = tensor(eye(30), destroy(30))
    n1 = dagger(a1) @ a1
    n2 = dagger(a2) @ a2
    h = (0.0 * (n1 + n2) + 1.0 * (dagger(a1) @ a2 + dagger(a2) @ a1)
         + 0.2 * (dagger(a1) @ dagger(a1) @ a1 @ a1 + dagger(a2) @ dagger(a2) @ a2 @ a2)
         + 0.5 * (a1 + dagger(a1)))
    ops = OperatorSet(h, (sqrt(0.2) * a1, sqrt(0.2) * a2), (n1, n2))
    return _problem(ops, fock(900, 0), 40.0, 400, log_jumps)


def stiff_cavity(log_jumps=True):
    """Stiff test case for the BDF fixtures (not a BASELINE config): a
    driven cavity, N=12, whose decay rate kappa=40 far exceeds the drive
    and detuning, t in [0, 5] with 101 output times."""
    a = destroy(12)
    ad = dagger(a)
    ops = OperatorSet(0.3 * (ad @ a) + 2.0 * (a + ad), (sqrt(40.0) * a,), (ad @ a, (a + ad) / 2))
    return _problem(ops, coherent(12, 1.0), 5.0, 100, log_jumps)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
