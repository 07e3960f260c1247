"""ctypes front end of the C oracle (TEST INFRASTRUCTURE / CPU BASELINE).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU leg may import
this module.  It runs the CPU restatement of the reference trajectory path
(oracle/mcwf_oracle.c) on the same packed problem the device receives and
returns per-trajectory results in the device engine's layout.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmcwf_oracle.so")

NSTATS = 16
STAT_NAMES = ("attempts", "steps", "corr_fail", "err_reject", "nfe", "corr_iters", "jumps",
              "bisect", "sum_q", "order_up", "order_down", "draws",
              "sum_qq1", "overflow_attempts",  # device-only counters (always 0 here)
              "lu_factor")
STREAM_KINDS = {"philox": 0, "lfsr113": 1, "scripted": 2}

_I64P = C.POINTER(C.c_int64)
_F64P = C.POINTER(C.c_double)


class MoCsr(C.Structure):
    _fields_ = [("row_ptr", _I64P), ("col_ind", _I64P), ("values", _F64P), ("nnz", C.c_int64)]


class MoProblem(C.Structure):
    _fields_ = [("dim", C.c_int64), ("g", MoCsr), ("n_collapse", C.c_int32),
                ("collapse", C.POINTER(MoCsr)), ("n_expect", C.c_int32),
                ("expect", C.POINTER(MoCsr)), ("psi0", _F64P), ("t_from", C.c_double),
                ("t_to", C.c_double), ("n_steps", C.c_int64), ("times", _F64P),
                ("rtol", C.c_double), ("atol", C.c_double), ("max_order", C.c_int32),
                ("max_steps", C.c_int64), ("h0_first", C.c_double), ("l_table", _F64P),
                ("tau1", _F64P), ("tau2", _F64P), ("tau3", _F64P), ("method", C.c_int32),
                ("n_td", C.c_int32), ("td", C.POINTER(MoCsr)), ("td_coef", _F64P)]


class MoRunArgs(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("traj_begin", C.c_int64), ("traj_end", C.c_int64),
                ("stream_kind", C.c_int32), ("script", _F64P), ("script_len", _I64P),
                ("script_stride", C.c_int64), ("script_fallback", C.c_double),
                ("max_jumps", C.c_int64), ("n_threads", C.c_int32),
                ("n_psi_points", C.c_int32), ("psi_points", _I64P)]


class MoError(C.Structure):
    _fields_ = [("code", C.c_int32), ("traj", C.c_int64), ("t", C.c_double), ("h", C.c_double),
                ("max_steps", C.c_int64), ("aux0", C.c_double), ("aux1", C.c_double),
                ("aux2", C.c_double)]


class MoRunOut(C.Structure):
    _fields_ = [("values", _F64P), ("stats", _I64P), ("status", C.POINTER(C.c_int32)),
                ("jump_count", _I64P), ("jump_t", _F64P), ("jump_idx", C.POINTER(C.c_int32)),
                ("error", MoError), ("psi", _F64P)]


_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "mcwf_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.mo_run.argtypes = [C.POINTER(MoProblem), C.POINTER(MoRunArgs), C.POINTER(MoRunOut)]
        _lib.mo_run.restype = C.c_int
        _lib.mo_philox_u01.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        _lib.mo_philox_u01.restype = C.c_double
        _lib.mo_lfsr113_derive.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint32)]
        _lib.mo_lfsr113_derive.restype = None
    return _lib


def _p(a, t=_F64P):
    return a.ctypes.data_as(t)


def _csr(m, keep):
    keep += [m.row_ptr, m.col_ind, m.values]
    return MoCsr(_p(m.row_ptr, _I64P), _p(m.col_ind, _I64P), _p(m.values), m.nnz)


def run(packed, seed: int, traj_begin: int, traj_end: int, *, stream: str = "philox",
        n_threads: int | None = None, script=None, script_fallback: float = 0.999999,
        max_jumps: int = 256, psi_points=None):
    """Run trajectories [traj_begin, traj_end) of a PackedProblem on the CPU.

    Returns a dict with ``values`` [n, n_expect, n_pts], ``stats`` [n, 16],
    ``status`` [n], ``jump_count`` [n], ``jump_t``/``jump_idx`` [n, max_jumps],
    ``psi`` [n, len(psi_points), dim] (complex, the state recorded at those
    grid indices; None without psi_points) and ``error`` (first failing
    trajectory, or None)."""
    L = lib()
    keep = []
    coll = (MoCsr * max(1, packed.n_collapse))(*[_csr(c, keep) for c in packed.collapse])
    expt = (MoCsr * max(1, packed.n_expect))(*[_csr(e, keep) for e in packed.expect])
    td = tuple(getattr(packed, "td", ()))
    tds = (MoCsr * max(1, len(td)))(*[_csr(m, keep) for m in td])
    td_coef = getattr(packed, "td_coef", None)
    prob = MoProblem(packed.dim, _csr(packed.g, keep), packed.n_collapse, coll,
                     packed.n_expect, expt, _p(packed.psi0), packed.t_from, packed.t_to,
                     packed.n_steps, _p(packed.times), packed.rtol, packed.atol,
                     packed.max_order, packed.max_steps, packed.h0_first,
                     _p(packed.l_table), _p(packed.tau1), _p(packed.tau2), _p(packed.tau3),
                     getattr(packed, "method", 0), len(td), tds,
                     _p(td_coef) if td_coef is not None else None)
    n = traj_end - traj_begin
    script_arr = script_len = None
    stride = 0
    if stream == "scripted":
        rows = [list(map(float, s)) for s in script]
        stride = max(1, max(len(r) for r in rows))
        script_arr = np.zeros((n, stride))
        script_len = np.zeros(n, np.int64)
        for i, r in enumerate(rows):
            script_arr[i, : len(r)] = r
            script_len[i] = len(r)
    pts = None if psi_points is None else np.ascontiguousarray(psi_points, dtype=np.int64)
    args = MoRunArgs(seed & 0xFFFFFFFFFFFFFFFF, traj_begin, traj_end, STREAM_KINDS[stream],
                     _p(script_arr) if script_arr is not None else None,
                     _p(script_len, _I64P) if script_len is not None else None, stride,
                     script_fallback, max_jumps,
                     n_threads if n_threads else (os.cpu_count() or 1),
                     0 if pts is None else len(pts), None if pts is None else _p(pts, _I64P))
    psi = None if pts is None else np.zeros((n, len(pts), packed.dim), dtype=np.complex128)
    values = np.zeros((n, packed.n_expect, packed.n_pts))
    stats = np.zeros((n, NSTATS), np.int64)
    status = np.zeros(n, np.int32)
    jcount = np.zeros(n, np.int64)
    jt = np.zeros((n, max_jumps))
    jidx = np.zeros((n, max_jumps), np.int32)
    out = MoRunOut(_p(values), _p(stats, _I64P), _p(status, C.POINTER(C.c_int32)),
                   _p(jcount, _I64P), _p(jt), _p(jidx, C.POINTER(C.c_int32)))
    out.psi = psi.view(np.float64).ctypes.data_as(_F64P) if psi is not None else None
    rc = L.mo_run(C.byref(prob), C.byref(args), C.byref(out))
    err = None
    if rc:
        e = out.error
        err = {"code": e.code, "traj": e.traj, "t": e.t, "h": e.h, "max_steps": e.max_steps,
               "aux": (e.aux0, e.aux1, e.aux2)}
    return {"values": values, "stats": stats, "status": status, "jump_count": jcount,
            "jump_t": jt, "jump_idx": jidx, "error": err, "rc": rc, "psi": psi}


def philox_u01(seed: int, k: int, n: int) -> float:
    return lib().mo_philox_u01(seed, k, n)


def lfsr113_words(seed: int, k: int):
    z = (C.c_uint32 * 4)()
    lib().mo_lfsr113_derive(seed, k, z)
    return tuple(z)
