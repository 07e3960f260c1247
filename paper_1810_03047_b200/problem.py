"""Boundary types of the trajectory path, mirroring the reference API.

The device engine takes a problem with the reference's field names
(``QuantumProblem``, /root/reference/pkg/src/mcwf/trajectory.py:46-103;
``OdeConfig``, ode.py:124-151) and returns a ``TrajectoryResult``
(trajectory.py:106-119).  A reference-built ``mcwf.QuantumProblem`` is
accepted as-is (duck typing on the same attributes), which is what makes
:func:`paper_1810_03047_b200.run_gpu` a drop-in for ``mcwf.run_inline``.

Also here: the Adams coefficient tables (restated from the generating
polynomials with exact rational arithmetic, ode.py:90-121) and the automatic
first step (ode.py:247-252), both computed once per problem on the host and
shipped to the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from math import sqrt

import numpy as np

from .csr import CsrMatrix, as_vector, csr_matvec, to_csr
from .qops import EffectiveGenerator, OperatorSet, effective_generator

__all__ = ["ADAMS", "BDF", "OdeConfig", "OdeFailure", "RunOptions", "QuantumProblem",
           "TrajectoryResult", "average_trajectories", "adams_tables", "bdf_tables",
           "method_tables", "auto_step", "LROWS"]

ADAMS = "adams"
BDF = "bdf"
_ORDER_LIMIT = {ADAMS: 12, BDF: 6}
LROWS = 13  # Nordsieck rows for Adams order <= 12


class OdeFailure(RuntimeError):
    """Integration halt with the reference's ISTATE code and message
    ("HALT: Error in ode solver, value ISTATE = ...", ode.py:53-62)."""

    def __init__(self, istate: int, detail: str):
        super().__init__(f"HALT: Error in ode solver, value ISTATE = {istate} ({detail})")
        self.istate = istate


@dataclass(frozen=True)
class OdeConfig:
    method: str = ADAMS
    rtol: float = 1e-7
    atol: float = 1e-12
    max_order: int | None = None
    max_steps: int = 50_000
    initial_step: float | None = None

    def __post_init__(self):
        if self.method not in _ORDER_LIMIT:
            raise ValueError(f"unknown method {self.method!r}")
        if not 0.0 < self.rtol < 1.0:
            raise ValueError("rtol must lie in (0, 1)")
        if self.atol < 0.0:
            raise ValueError("atol must be non-negative")
        limit = _ORDER_LIMIT[self.method]
        if self.max_order is None:
            object.__setattr__(self, "max_order", limit)
        elif not 1 <= self.max_order <= limit:
            raise ValueError(f"max_order must be in [1, {limit}] for {self.method}")
        if self.max_steps < 1:
            raise ValueError("max_steps must be positive")
        if self.initial_step is not None and self.initial_step <= 0:
            raise ValueError("initial_step must be positive")


@dataclass(frozen=True)
class RunOptions:
    only_final_trj: bool = True
    output_target: str = "-"
    verbose: bool = False
    log_jumps: bool = False


@dataclass(frozen=True)
class QuantumProblem:
    generator: EffectiveGenerator | None
    collapse_csr: tuple
    expect_csr: tuple
    psi0: np.ndarray
    t_from: float
    t_to: float
    n_steps: int
    ode: OdeConfig = field(default_factory=OdeConfig)
    options: RunOptions = field(default_factory=RunOptions)
    rhs_fn: object = None

    def __post_init__(self):
        psi0 = as_vector(self.psi0)
        object.__setattr__(self, "psi0", psi0)
        object.__setattr__(self, "collapse_csr", tuple(self.collapse_csr))
        object.__setattr__(self, "expect_csr", tuple(self.expect_csr))
        if not np.all(np.isfinite(psi0.view(np.float64))):
            raise ValueError("psi0 must be finite")
        if abs(float(np.vdot(psi0, psi0).real) - 1.0) > 1e-12:
            raise ValueError("psi0 must be normalised to 1 within 1e-12")
        if (self.generator is None) == (self.rhs_fn is None):
            raise ValueError("exactly one of generator / rhs_fn must be given")
        dim = psi0.shape[0]
        if self.generator is not None and self.generator.dim != dim:
            raise ValueError(f"generator dim {self.generator.dim} != state dim {dim}")
        for m in (*self.collapse_csr, *self.expect_csr):
            if getattr(m, "n", None) != dim:
                raise ValueError("collapse/expect operators must be CSR of the state dim")
        if not self.t_to > self.t_from:
            raise ValueError("t_to must exceed t_from")
        if self.n_steps < 1:
            raise ValueError("n_steps must be positive")

    @property
    def dim(self) -> int:
        return self.psi0.shape[0]

    def time_grid(self) -> np.ndarray:
        return np.linspace(self.t_from, self.t_to, self.n_steps + 1)

    @classmethod
    def from_operators(cls, ops: OperatorSet, psi0, t_from, t_to, n_steps,
                       ode: OdeConfig | None = None,
                       options: RunOptions | None = None) -> "QuantumProblem":
        return cls(generator=effective_generator(ops),
                   collapse_csr=tuple(to_csr(c) for c in ops.collapse),
                   expect_csr=tuple(to_csr(e) for e in ops.expect),
                   psi0=psi0, t_from=float(t_from), t_to=float(t_to), n_steps=int(n_steps),
                   ode=ode if ode is not None else OdeConfig(),
                   options=options if options is not None else RunOptions())


@dataclass(frozen=True)
class TrajectoryResult:
    """Expectation-value series averaged over ``n_trajectories`` runs.

    ``sumsq`` (optional, device engine only) carries the per-point sum of
    squares over trajectories so callers can form standard errors."""

    times: np.ndarray
    values: np.ndarray
    n_trajectories: int
    jumps: list | None = None
    sumsq: np.ndarray | None = None
    stats: dict | None = None

    def __post_init__(self):
        object.__setattr__(self, "times", np.ascontiguousarray(self.times, dtype=np.float64))
        object.__setattr__(self, "values", np.ascontiguousarray(self.values, dtype=np.float64))
        if self.values.ndim != 2 or self.values.shape[1] != self.times.shape[0]:
            raise ValueError("values must be (n_expect, n_times)")

    def standard_error(self) -> np.ndarray:
        if self.sumsq is None or self.n_trajectories < 2:
            raise ValueError("standard error needs sumsq and >= 2 trajectories")
        n = self.n_trajectories
        var = (self.sumsq / n - self.values ** 2) * n / (n - 1)
        return np.sqrt(np.maximum(var, 0.0) / n)


def average_trajectories(results) -> TrajectoryResult:
    """Count-weighted mean of partial results on one grid (same contract as
    the reference, trajectory.py:253-273)."""
    results = list(results)
    if not results:
        raise ValueError("nothing to average")
    first = results[0]
    total = 0
    acc = np.zeros_like(first.values)
    jumps = [] if all(r.jumps is not None for r in results) else None
    for r in results:
        if r.values.shape != first.values.shape or not np.array_equal(r.times, first.times):
            raise ValueError("trajectory results have mismatching grids")
        if r.n_trajectories:
            acc += r.n_trajectories * r.values
        total += r.n_trajectories
        if jumps is not None:
            jumps.extend(r.jumps)
    if total > 0:
        acc /= total
    return TrajectoryResult(first.times, acc, total, jumps)


# -- Adams coefficients ---------------------------------------------------------


def _adams_rational(max_order: int = 12):
    """Adams-Moulton Nordsieck vectors l(q), error constants tau2(q), from
    p_q(x) = prod_{i=1}^{q-1} (x + i):  l0 = int_{-1}^0 p / (q-1)!,  l1 = 1,
    l_j = [x^{j-1}]p / (j (q-1)!),  tau2 = q! / |int_{-1}^0 x p|."""
    def integral(coeffs, extra_power):
        return sum(c * Fraction((-1) ** (i + extra_power), i + extra_power + 1)
                   for i, c in enumerate(coeffs))

    poly = [Fraction(1)]
    fact = Fraction(1)  # (q-1)!
    rows = {}
    for q in range(1, max_order + 1):
        if q > 1:
            fact *= q - 1
        l = [integral(poly, 0) / fact, Fraction(1)]
        l += [poly[j - 1] / (j * fact) for j in range(2, q + 1)]
        tau2 = (fact * q) / abs(integral(poly, 1))
        rows[q] = (l, tau2)
        nxt = [Fraction(0)] * (len(poly) + 1)  # multiply by (x + q)
        for i, c in enumerate(poly):
            nxt[i] += c * q
            nxt[i + 1] += c
        poly = nxt
    return rows


def adams_tables(max_order: int = 12):
    """Float tables: ``l[q, 0..q]``, ``tau1[q]`` (order-down divisor,
    tau2(q-1)/q!), ``tau2[q]``, ``tau3[q]`` (order-up divisor, tau2(q+1)),
    all indexed by order q = 1..12 (row/entry 0 unused)."""
    rows = _adams_rational(max_order)
    l_tab = np.zeros((LROWS, LROWS))
    tau1 = np.zeros(LROWS)
    tau2 = np.zeros(LROWS)
    tau3 = np.zeros(LROWS)
    qfact = 1.0
    for q in range(1, max_order + 1):
        l, t2 = rows[q]
        l_tab[q, : q + 1] = [float(c) for c in l]
        tau2[q] = float(t2)
    for q in range(2, max_order + 1):
        qfact = float(np.prod(np.arange(1, q + 1, dtype=np.float64)))
        tau1[q] = tau2[q - 1] / qfact
    for q in range(1, max_order):
        tau3[q] = tau2[q + 1]
    return l_tab, tau1, tau2, tau3


def bdf_tables(max_order: int = 6):
    """BDF Nordsieck vectors and error divisors (ode.py:108-119), from
    P_q(x) = (x+1)(x+2)...(x+q) in exact rationals: l_j = [x^j]P / [x^1]P,
    H_q = [x^1]P / [x^0]P, tau2 = (q+1) H_q (same order), tau3 = (q+2) H_q
    (order up), tau1 = 1/(q-1)! (order down, q >= 2).  Same table layout as
    :func:`adams_tables` (rows 7..12 unused)."""
    l_tab = np.zeros((LROWS, LROWS))
    tau1 = np.zeros(LROWS)
    tau2 = np.zeros(LROWS)
    tau3 = np.zeros(LROWS)
    poly = [Fraction(1)]
    for q in range(1, max_order + 1):
        nxt = [Fraction(0)] * (len(poly) + 1)  # multiply by (x + q)
        for i, c in enumerate(poly):
            nxt[i] += c * q
            nxt[i + 1] += c
        poly = nxt
        l_tab[q, : q + 1] = [float(c / poly[1]) for c in poly]
        hq = poly[1] / poly[0]
        tau2[q] = float((q + 1) * hq)
        tau3[q] = float((q + 2) * hq)
        if q >= 2:
            fact = Fraction(1)
            for i in range(2, q):
                fact *= i
            tau1[q] = 1.0 / float(fact)
    return l_tab, tau1, tau2, tau3


def method_tables(method: str):
    """(l, tau1, tau2, tau3) of the ODE method family."""
    if method == ADAMS:
        return adams_tables()
    if method == BDF:
        return bdf_tables()
    raise ValueError(f"unknown method {method!r}")


def auto_step(g, y0: np.ndarray, rtol: float, atol: float, f0=None) -> float:
    """Automatic first step h = 0.01 / ||G y0||_wrms with weights
    1/(atol + rtol |y0_i|) (ode.py:247-252), evaluated with the same numpy
    expression (a BLAS dot) as the reference so the value matches it.
    ``f0`` overrides G y0 (a time-dependent right side at t_from)."""
    if f0 is None:
        f0 = csr_matvec(g, y0)
    w2 = 1.0 / (atol + rtol * np.abs(y0)) ** 2
    fw = sqrt(float((f0.real * f0.real + f0.imag * f0.imag) @ w2) / y0.shape[0])
    if fw <= 0.0:
        return 1e-6
    return 0.01 / fw


# -- the reference's own result / exception types at the boundary ---------------

_REF_TYPES: dict = {}


def _reference_module(problem=None):
    """The reference package ``mcwf`` when the caller uses it: the problem
    is an ``mcwf`` object, or ``mcwf`` is already imported.  (Never imported
    just for this -- the device path does not depend on the reference.)"""
    import sys
    mod = type(problem).__module__.split(".")[0] if problem is not None else ""
    if mod == "mcwf" or "mcwf" in sys.modules:
        try:
            import mcwf  # noqa: F401
            import mcwf.ode
            import mcwf.trajectory
            return sys.modules["mcwf"]
        except ImportError:
            return None
    return None


def reference_types(problem=None):
    """``(OdeFailure, TrajectoryResult)`` classes for results handed back to
    the caller.  With ``mcwf`` in use they are subclasses of BOTH the
    reference's classes (``mcwf.ode.OdeFailure``, ode.py:53-62, and
    ``mcwf.trajectory.TrajectoryResult``, trajectory.py:106-119) and this
    package's mirrors, so ``except mcwf.OdeFailure`` and
    ``isinstance(r, mcwf.TrajectoryResult)`` hold for device results while
    ``sumsq`` / ``stats`` / ``standard_error()`` stay available."""
    mc = _reference_module(problem)
    if mc is None:
        return OdeFailure, TrajectoryResult
    key = id(mc)
    if key not in _REF_TYPES:
        from dataclasses import dataclass as _dc

        class DeviceOdeFailure(mc.ode.OdeFailure, OdeFailure):
            __module__ = __name__

            def __init__(self, istate: int, detail: str):
                RuntimeError.__init__(
                    self, f"HALT: Error in ode solver, value ISTATE = {istate} ({detail})")
                self.istate = istate

        @_dc(frozen=True)
        class DeviceTrajectoryResult(mc.trajectory.TrajectoryResult, TrajectoryResult):
            __module__ = __name__

        DeviceOdeFailure.__qualname__ = DeviceOdeFailure.__name__ = "OdeFailure"
        DeviceTrajectoryResult.__qualname__ = DeviceTrajectoryResult.__name__ = "TrajectoryResult"
        _REF_TYPES[key] = (DeviceOdeFailure, DeviceTrajectoryResult)
    return _REF_TYPES[key]
