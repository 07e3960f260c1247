"""ctypes binding of libqtm.so (include/qtm.h).

The shared library is built in-tree by ``paper_1810_03047_b200.build``.
There is no CPU fallback: if the library is missing or cannot be loaded,
:func:`lib` raises, and every device entry point fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QTM_LIB") or os.path.join(HERE, "libqtm.so")

ABI_VERSION = 3
BLOCK = 256  # QTM_BLOCK: trajectories per fixed-order reduction block
NSTATS = 16
LROWS = 13
MAX_OPS = 32

STREAM_KINDS = {"philox": 0, "lfsr113": 1, "scripted": 2}
STAT_NAMES = ("attempts", "steps", "corr_fail", "err_reject", "nfe", "corr_iters", "jumps",
              "bisect", "sum_q", "order_up", "order_down", "draws", "sum_qq1",
              "overflow_attempts", "lu_factor")

# status codes (enum qtm_status)
OK = 0
ERR_MAX_STEPS = -1
ERR_REPEATED_ERRTEST = -4
ERR_STEP_COLLAPSE = -5
ERR_CORRECTOR = -6
ERR_BRACKET = -10
ERR_NO_SUPPORT = -11
ERR_ZERO_VECTOR = -12
ERR_ARGS = -20
ERR_CUDA = -21
ERR_UNSUPPORTED = -22

_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)
_F64P = C.POINTER(C.c_double)


class QtmCsr(C.Structure):
    _fields_ = [("row_ptr", _I64P), ("col_ind", _I64P), ("values", _F64P), ("nnz", C.c_int64)]


class QtmProblemDesc(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("dim", C.c_int64), ("generator", QtmCsr),
                ("n_collapse", C.c_int32), ("collapse", C.POINTER(QtmCsr)),
                ("n_expect", C.c_int32), ("expect", C.POINTER(QtmCsr)), ("psi0", _F64P),
                ("t_from", C.c_double), ("t_to", C.c_double), ("n_steps", C.c_int64),
                ("times", _F64P), ("method", C.c_int32), ("rtol", C.c_double),
                ("atol", C.c_double), ("max_order", C.c_int32), ("max_steps", C.c_int64),
                ("h0_first", C.c_double), ("l_table", _F64P), ("tau1", _F64P), ("tau2", _F64P),
                ("tau3", _F64P), ("device", C.c_int32), ("variant", C.c_int32),
                ("n_td", C.c_int32), ("td", C.POINTER(QtmCsr)), ("td_coef", _F64P)]


class QtmRunArgs(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("traj_begin", C.c_int64), ("traj_end", C.c_int64),
                ("stream_kind", C.c_int32), ("script", _F64P), ("script_len", _I64P),
                ("script_stride", C.c_int64), ("script_fallback", C.c_double),
                ("max_jumps", C.c_int64), ("cuda_stream", C.c_void_p),
                ("n_psi_points", C.c_int32), ("psi_points", _I64P)]


class QtmError(C.Structure):
    _fields_ = [("code", C.c_int32), ("traj", C.c_int64), ("t", C.c_double), ("h", C.c_double),
                ("max_steps", C.c_int64), ("aux0", C.c_double), ("aux1", C.c_double),
                ("aux2", C.c_double)]


class QtmRunOut(C.Structure):
    _fields_ = [("sum", _F64P), ("sumsq", _F64P), ("values", _F64P), ("stats", _I64P),
                ("stats_total", _I64P), ("status", _I32P), ("jump_count", _I64P),
                ("jump_t", _F64P), ("jump_idx", _I32P), ("error", QtmError),
                ("kernel_ms", C.c_float), ("total_ms", C.c_float), ("variant", C.c_int32),
                ("grid", C.c_int32), ("launches", C.c_int64), ("n_failed", C.c_int64),
                ("psi", _F64P), ("block_sum", _F64P), ("block_sumsq", _F64P)]


EXPORTS = ("qtm_problem_create", "qtm_run", "qtm_run_resident", "qtm_problem_destroy",
           "qtm_max_resident", "qtm_problem_layout",
           "qtm_last_error", "qtm_abi_version", "qtm_num_variants", "qtm_variant_info",
           "qtm_device_count", "qtm_measure_fp64_peak", "qtm_phase_cycles",
           "qtm_variant_time_dependent", "qtm_measure_dmma_peak", "qtm_variant_tmem_rows",
           "qtm_problem_variant", "qtm_variant_small")

_lib = None


class NativeLibraryError(ImportError):
    pass


def lib():
    """Load libqtm.so (raises NativeLibraryError if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not found: build it with `python -m paper_1810_03047_b200.build` "
            "(there is no CPU fallback for the trajectory engine)")
    L = C.CDLL(LIB_PATH)
    L.qtm_problem_create.argtypes = [C.POINTER(QtmProblemDesc), C.POINTER(C.c_void_p)]
    L.qtm_problem_create.restype = C.c_int
    L.qtm_run.argtypes = [C.c_void_p, C.POINTER(QtmRunArgs), C.POINTER(QtmRunOut)]
    L.qtm_run.restype = C.c_int
    L.qtm_run_resident.argtypes = [C.c_void_p, C.POINTER(QtmRunArgs), C.POINTER(QtmRunOut)]
    L.qtm_run_resident.restype = C.c_int
    L.qtm_max_resident.argtypes = [C.c_void_p, _I32P]
    L.qtm_max_resident.restype = C.c_int
    L.qtm_problem_layout.argtypes = [C.c_void_p, _I32P, _I32P, C.POINTER(C.c_int64)]
    L.qtm_problem_layout.restype = C.c_int
    L.qtm_problem_destroy.argtypes = [C.c_void_p]
    L.qtm_problem_destroy.restype = None
    L.qtm_last_error.argtypes = []
    L.qtm_last_error.restype = C.c_char_p
    L.qtm_abi_version.argtypes = []
    L.qtm_abi_version.restype = C.c_int
    L.qtm_num_variants.argtypes = []
    L.qtm_num_variants.restype = C.c_int
    L.qtm_variant_info.argtypes = [C.c_int, _I32P, _I32P, _I32P]
    L.qtm_variant_info.restype = C.c_int
    L.qtm_variant_time_dependent.argtypes = [C.c_int]
    L.qtm_variant_time_dependent.restype = C.c_int
    L.qtm_variant_small.argtypes = [C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.qtm_variant_small.restype = C.c_int
    L.qtm_problem_variant.argtypes = [C.c_void_p]
    L.qtm_problem_variant.restype = C.c_int
    L.qtm_variant_tmem_rows.argtypes = [C.c_int]
    L.qtm_variant_tmem_rows.restype = C.c_int
    L.qtm_device_count.argtypes = []
    L.qtm_device_count.restype = C.c_int
    if hasattr(L, "qtm_phase_cycles"):
        L.qtm_phase_cycles.argtypes = [C.POINTER(C.c_uint64)]
        L.qtm_phase_cycles.restype = C.c_int
    L.qtm_measure_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    L.qtm_measure_fp64_peak.restype = C.c_int
    L.qtm_measure_dmma_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    L.qtm_measure_dmma_peak.restype = C.c_int
    if L.qtm_abi_version() != ABI_VERSION:
        raise NativeLibraryError("libqtm.so ABI version mismatch; rebuild it")
    _lib = L
    return L


def last_error() -> str:
    return lib().qtm_last_error().decode(errors="replace")


def variants():
    L = lib()
    out = []
    for i in range(L.qtm_num_variants()):
        t, e, r = C.c_int32(), C.c_int32(), C.c_int32()
        L.qtm_variant_info(i, C.byref(t), C.byref(e), C.byref(r))
        out.append((t.value, e.value, r.value))
    return out


def dmma_peak_tflops(device: int = 0) -> float:
    out = C.c_double()
    rc = lib().qtm_measure_dmma_peak(device, C.byref(out))
    if rc != 0:
        raise RuntimeError(f"qtm_measure_dmma_peak failed: {last_error()}")
    return out.value


def variant_time_dependent(i: int) -> bool:
    return lib().qtm_variant_time_dependent(i) == 1


def variant_small(i: int) -> tuple[int, int]:
    """(d_max, trajectories per warp) of a one-thread-per-trajectory variant,
    (0, 0) for the CTA-per-trajectory variants."""
    dm, ln = C.c_int32(), C.c_int32()
    if lib().qtm_variant_small(i, C.byref(dm), C.byref(ln)) != 0:
        raise RuntimeError(last_error())
    return dm.value, ln.value


def variant_tmem_rows(i: int) -> int:
    """Nordsieck rows the variant keeps in Tensor Memory (0: none)."""
    return max(0, lib().qtm_variant_tmem_rows(i))


def fp64_peak_tflops(device: int = 0) -> float:
    out = C.c_double()
    rc = lib().qtm_measure_fp64_peak(device, C.byref(out))
    if rc != 0:
        raise RuntimeError(f"qtm_measure_fp64_peak failed: {last_error()}")
    return out.value


PHASES = ("step-level", "predict", "gather", "spmv", "update", "reduction", "convergence",
          "error-test/commit", "order-control", "jump-test/jumps", "recording", "accept+weights")


def phase_cycles():
    arr = (C.c_uint64 * 16)()
    lib().qtm_phase_cycles(arr)
    return {name: int(arr[i]) for i, name in enumerate(PHASES)}
