"""Flatten a ``QuantumProblem`` into the plain arrays the C-ABI takes.

The device boundary (include/qtm.h) receives CSR operators as
(int64 row_ptr, int64 col_ind, float64 interleaved (re, im) values) -- the
reference's own ``CsrMatrix`` layout (linalg.py:43-60) viewed as float64 --
plus psi0, the output grid from ``np.linspace`` (trajectory.py:89-90), the
ODE configuration, the Adams tables and the first-segment step size.
"""

from __future__ import annotations

from dataclasses import dataclass
from hashlib import blake2b

import numpy as np

from .problem import ADAMS, BDF, auto_step, method_tables

__all__ = ["PackedCsr", "PackedProblem", "pack_problem"]


@dataclass(frozen=True)
class PackedCsr:
    n: int
    row_ptr: np.ndarray  # int64 [n+1]
    col_ind: np.ndarray  # int64 [nnz]
    values: np.ndarray   # float64 [2*nnz] interleaved

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @classmethod
    def from_csr(cls, m) -> "PackedCsr":
        vals = np.ascontiguousarray(np.asarray(m.values, dtype=np.complex128)).view(np.float64)
        return cls(int(m.n), np.ascontiguousarray(m.row_ptr, dtype=np.int64),
                   np.ascontiguousarray(m.col_ind, dtype=np.int64), np.ascontiguousarray(vals))


@dataclass(frozen=True)
class PackedProblem:
    dim: int
    g: PackedCsr
    collapse: tuple
    expect: tuple
    psi0: np.ndarray      # float64 [2*dim]
    t_from: float
    t_to: float
    n_steps: int
    times: np.ndarray     # float64 [n_steps+1]
    rtol: float
    atol: float
    max_order: int
    max_steps: int
    h0_first: float
    l_table: np.ndarray   # float64 [13*13]
    tau1: np.ndarray
    tau2: np.ndarray
    tau3: np.ndarray
    log_jumps: bool
    digest: int
    method: int = 0        # 0 = ADAMS, 1 = BDF (qtm_problem_desc.method)
    td: tuple = ()         # time-dependent terms G_k (PackedCsr), timedep.py
    td_coef: np.ndarray | None = None  # float64 [n_td*4]: amp, omega, phase, offset

    @property
    def n_expect(self) -> int:
        return len(self.expect)

    @property
    def n_collapse(self) -> int:
        return len(self.collapse)

    @property
    def n_pts(self) -> int:
        return self.n_steps + 1

    @property
    def n_td(self) -> int:
        return len(self.td)

    def nbytes(self) -> int:
        total = self.psi0.nbytes + self.times.nbytes
        for m in (self.g, *self.collapse, *self.expect, *self.td):
            total += m.row_ptr.nbytes + m.col_ind.nbytes + m.values.nbytes
        return total


def _digest(parts) -> int:
    h = blake2b(digest_size=8)
    for p in parts:
        h.update(np.ascontiguousarray(p).tobytes() if isinstance(p, np.ndarray) else repr(p).encode())
    return int.from_bytes(h.digest(), "little")


def pack_problem(problem, *, h0_first: float | None = None) -> PackedProblem:
    """Validate and flatten.  The device integrates a constant generator
    with either method family: ADAMS (the numba kernel path,
    _kernels.py:117-192) or BDF (modified Newton with a dense LU of
    I - h l0 G, ode.py:334-423); the l/tau tables follow the method."""
    from .timedep import TimeDependentGenerator
    ode = problem.ode
    if ode.method not in (ADAMS, BDF):
        raise ValueError(f"unknown ODE method {ode.method!r}")
    gen = getattr(problem, "generator", None)
    rhs = getattr(problem, "rhs_fn", None)
    td, td_coef = (), None
    if gen is not None:
        g0 = gen.g
    elif isinstance(rhs, TimeDependentGenerator):
        # H(t) = H0 + sum_k c_k(t) H_k on the device (timedep.py); the general
        # engine integrates it with the Adams functional corrector
        # (ode.py:227-230, 358-377) -- BDF would need finite-difference
        # Jacobians of the callback (ode.py:425-437), not on the device
        if ode.method != ADAMS:
            raise ValueError("time-dependent generators run with the ADAMS method only")
        g0 = rhs.g0
        td = tuple(PackedCsr.from_csr(m) for m, _ in rhs.terms)
        td_coef = np.ascontiguousarray(np.concatenate([c.as_array() for _, c in rhs.terms]))
    else:
        raise ValueError("device engine needs a constant generator or a TimeDependentGenerator "
                         "rhs_fn (an arbitrary rhs_fn callback cannot run on the GPU)")
    g = PackedCsr.from_csr(g0)
    psi0 = np.ascontiguousarray(np.asarray(problem.psi0, dtype=np.complex128))
    dim = psi0.shape[0]
    if g.n != dim:
        raise ValueError(f"generator dim {g.n} != state dim {dim}")
    collapse = tuple(PackedCsr.from_csr(c) for c in problem.collapse_csr)
    expect = tuple(PackedCsr.from_csr(e) for e in problem.expect_csr)
    for m in (*collapse, *expect, *td):
        if m.n != dim:
            raise ValueError("collapse/expect operators must be CSR of the state dim")
    times = np.linspace(problem.t_from, problem.t_to, problem.n_steps + 1)
    if h0_first is None:
        h0_first = ode.initial_step if ode.initial_step is not None else \
            auto_step(g0, psi0, ode.rtol, ode.atol,
                      f0=None if not td else np.asarray(rhs(problem.t_from, psi0), np.complex128))
    l_tab, tau1, tau2, tau3 = method_tables(ode.method)
    log_jumps = bool(getattr(getattr(problem, "options", None), "log_jumps", False))
    digest = _digest([dim, g.row_ptr, g.col_ind, g.values,
                      *[a for m in (*collapse, *expect) for a in (m.row_ptr, m.col_ind, m.values)],
                      len(collapse), len(expect), psi0, problem.t_from, problem.t_to,
                      problem.n_steps, ode.rtol, ode.atol, ode.max_order, ode.max_steps,
                      float(h0_first)] + ([ode.method] if ode.method != ADAMS else [])
                     + [a for m in td for a in (m.row_ptr, m.col_ind, m.values)]
                     + ([td_coef] if td else []))
    return PackedProblem(dim=dim, g=g, collapse=collapse, expect=expect,
                         psi0=psi0.view(np.float64).copy(), t_from=float(problem.t_from),
                         t_to=float(problem.t_to), n_steps=int(problem.n_steps), times=times,
                         rtol=float(ode.rtol), atol=float(ode.atol),
                         max_order=int(ode.max_order), max_steps=int(ode.max_steps),
                         h0_first=float(h0_first), l_table=np.ascontiguousarray(l_tab.ravel()),
                         tau1=tau1, tau2=tau2, tau3=tau3, log_jumps=log_jumps, digest=digest,
                         method=0 if ode.method == ADAMS else 1, td=td, td_coef=td_coef)
