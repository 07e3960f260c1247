"""Time-dependent Hamiltonians on the device: H(t) = H0 + sum_k c_k(t) H_k.

The reference takes a time-dependent right side as an arbitrary callback,
``QuantumProblem(generator=None, rhs_fn=f)`` with ``f(t, psi) -> dpsi``
(trajectory.py:61, 72-73, 186; integrated by the general engine,
ode.py:227-230, 334-377).  A Python callback cannot run inside a GPU kernel,
so the device takes the structured form of the common case instead:

    psi' = G(t) psi,   G(t) = G0 + sum_k c_k(t) G_k,
    G0 = -i H0 - 1/2 sum_n C_n^+ C_n,   G_k = -i H_k,
    c_k(t) = offset_k + amp_k cos(omega_k t + phase_k).

:class:`TimeDependentGenerator` is that form AND a plain callable with the
reference's ``rhs_fn`` signature: handed to the reference's own
``QuantumProblem`` it runs on the CPU through the reference's general engine
(that is how the golden fixtures for this path were produced), and handed to
:func:`paper_1810_03047_b200.run_gpu` it is packed for the device.  The call
computes ``G0 psi`` and then adds ``c_k(t) * (G_k psi)`` term by term, the
order the device kernel uses.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .csr import CsrMatrix, as_matrix, csr_matvec, to_csr
from .qops import OperatorSet, effective_generator

__all__ = ["Coefficient", "TimeDependentGenerator", "MAX_TD_TERMS"]

MAX_TD_TERMS = 8  # include/qtm.h QTM_MAX_TD_TERMS


@dataclass(frozen=True)
class Coefficient:
    """c(t) = offset + amp * cos(omega * t + phase)  (sin: phase = -pi/2)."""

    amp: float
    omega: float = 0.0
    phase: float = 0.0
    offset: float = 0.0

    def __call__(self, t: float) -> float:
        return self.offset + self.amp * math.cos(self.omega * t + self.phase)

    def as_array(self) -> np.ndarray:
        return np.array([self.amp, self.omega, self.phase, self.offset], dtype=np.float64)


class TimeDependentGenerator:
    """psi' = (G0 + sum_k c_k(t) G_k) psi, usable as a reference ``rhs_fn``."""

    def __init__(self, g0: CsrMatrix, terms):
        self.g0 = g0
        self.terms = tuple((m, c if isinstance(c, Coefficient) else Coefficient(*c))
                           for m, c in terms)
        if not 1 <= len(self.terms) <= MAX_TD_TERMS:
            raise ValueError(f"between 1 and {MAX_TD_TERMS} time-dependent terms are supported")
        for m, _ in self.terms:
            if not isinstance(m, CsrMatrix) or m.n != g0.n:
                raise ValueError("time-dependent terms must be CsrMatrix of the state dim")

    @property
    def dim(self) -> int:
        return self.g0.n

    @classmethod
    def from_operators(cls, ops: OperatorSet, h_terms) -> "TimeDependentGenerator":
        """G0 from the static Hamiltonian and the collapse operators (as
        operators.py:116-126), plus G_k = -i H_k for each (H_k, c_k)."""
        g0 = effective_generator(ops).g
        terms = [(to_csr(-1j * as_matrix(h)), c) for h, c in h_terms]
        return cls(g0, terms)

    def __call__(self, t: float, psi: np.ndarray) -> np.ndarray:
        out = csr_matvec(self.g0, psi)
        for m, c in self.terms:
            out = out + c(t) * csr_matvec(m, psi)
        return out

