"""Host-side operator containers (setup time only, never on the hot path).

Mirrors the reference's ``mcwf.linalg`` surface that the trajectory path
consumes (/root/reference/pkg/src/mcwf/linalg.py:43-85, 111-133):
a square complex CSR matrix with int64 ``row_ptr``/``col_ind``, complex128
``values`` and strictly increasing columns per row.  Any object with those
four attributes (including the reference's own ``CsrMatrix``) is accepted by
the device boundary, so a reference-built problem drops in unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass
import numpy as np

__all__ = ["CsrMatrix", "as_vector", "as_matrix", "dagger", "tensor", "to_csr", "csr_matvec"]


def as_vector(data) -> np.ndarray:
    v = np.ascontiguousarray(data, dtype=np.complex128)
    if v.ndim != 1 or v.shape[0] < 1:
        raise ValueError(f"expected a 1-d vector of positive length, got shape {v.shape}")
    return v


def as_matrix(data) -> np.ndarray:
    m = np.ascontiguousarray(data, dtype=np.complex128)
    if m.ndim != 2 or m.shape[0] != m.shape[1] or m.shape[0] < 1:
        raise ValueError(f"expected a square matrix, got shape {m.shape}")
    return m


@dataclass(frozen=True)
class CsrMatrix:
    """Square complex CSR matrix (same field names as the reference)."""

    n: int
    row_ptr: np.ndarray
    col_ind: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        rp = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(self.col_ind, dtype=np.int64)
        va = np.ascontiguousarray(self.values, dtype=np.complex128)
        object.__setattr__(self, "row_ptr", rp)
        object.__setattr__(self, "col_ind", ci)
        object.__setattr__(self, "values", va)
        if self.n < 1:
            raise ValueError("CsrMatrix dimension must be positive")
        if rp.shape[0] != self.n + 1 or rp[0] != 0 or np.any(np.diff(rp) < 0):
            raise ValueError("row_ptr must be non-decreasing, start at 0 and have n+1 entries")
        if ci.shape[0] != rp[-1] or va.shape[0] != rp[-1]:
            raise ValueError("col_ind/values length must equal row_ptr[n]")
        if ci.size:
            if ci.min() < 0 or ci.max() >= self.n:
                raise ValueError("column index out of range")
            row_of = np.repeat(np.arange(self.n), np.diff(rp))
            same_row = row_of[1:] == row_of[:-1]
            if np.any(same_row & (np.diff(ci) <= 0)):
                raise ValueError("column indices not strictly increasing within a row")

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n), dtype=np.complex128)
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        out[rows, self.col_ind] = self.values
        return out


def dagger(m) -> np.ndarray:
    return np.ascontiguousarray(as_matrix(m).conj().T)


def tensor(*factors) -> np.ndarray:
    """Kronecker product; the first factor is the most significant index."""
    if not factors:
        raise ValueError("tensor() needs at least one factor")
    out = np.asarray(factors[0], dtype=np.complex128)
    for f in factors[1:]:
        out = np.kron(out, np.asarray(f, dtype=np.complex128))
    return out


def to_csr(m, drop_tol: float = 0.0) -> CsrMatrix:
    """Compress a dense matrix keeping entries with |value| > drop_tol, in
    row-major order (columns ascending within a row)."""
    if drop_tol < 0:
        raise ValueError("drop_tol must be non-negative")
    m = as_matrix(m)
    keep = np.abs(m) > drop_tol
    rows, cols = np.nonzero(keep)
    row_ptr = np.zeros(m.shape[0] + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    np.cumsum(row_ptr, out=row_ptr)
    return CsrMatrix(m.shape[0], row_ptr, cols.astype(np.int64), m[rows, cols])


def csr_matvec(m, x: np.ndarray) -> np.ndarray:
    """y = M x with every row summed left to right and each complex product
    formed as (ac - bd, ad + bc) without fused multiply-add -- the order of
    the reference's numba kernel (_kernels.py:19-27).  Vectorised over rows;
    numpy's own complex multiply is not used because its SIMD loop fuses."""
    x = as_vector(x)
    rp = np.asarray(m.row_ptr)
    ci = np.asarray(m.col_ind)
    va = np.asarray(m.values)
    n = x.shape[0]
    lens = np.diff(rp)
    acc_re = np.zeros(n)
    acc_im = np.zeros(n)
    xr, xi = x.real, x.imag
    for k in range(int(lens.max()) if n else 0):
        rows = np.nonzero(lens > k)[0]
        idx = rp[rows] + k
        a, b = va.real[idx], va.imag[idx]
        c, d = xr[ci[idx]], xi[ci[idx]]
        acc_re[rows] = acc_re[rows] + (a * c - b * d)
        acc_im[rows] = acc_im[rows] + (a * d + b * c)
    return acc_re + 1j * acc_im
