"""Device trajectory engine: the drop-in for the reference's trajectory loop.

``run_gpu(problem, n_total, master_seed)`` has the positional signature and
the return type of the reference's ``run_inline``
(/root/reference/pkg/src/mcwf/cluster.py:472-482): it integrates trajectories
0..n_total-1, averages ⟨E_k⟩(t_j) over them and returns a
``TrajectoryResult``.  The per-trajectory work (run_single_trajectory,
trajectory.py:190-250, and the solver it drives, ode.py) runs inside one
persistent sm_100a kernel per call behind the C ABI in include/qtm.h:
csrc/qtm_traj.cuh for the ADAMS family (constant generator, or a
TimeDependentGenerator rhs_fn, timedep.py), csrc/qtm_bdf.cuh for BDF.

Random streams are per trajectory and keyed by the global index (see
csrc/qtm_rng.cuh), so the ensemble does not depend on how it is sharded
over GPUs; the reference's single sequential per-worker stream cannot be
reproduced in parallel.

``run_sharded`` is the multi-GPU form (one process per GPU): contiguous
trajectory ranges per rank (partition_trajectories rule, cluster.py:369-377)
and one all-reduce of the per-point sums.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass

import numpy as np

from . import native
from .packing import PackedProblem, pack_problem
from .problem import OdeFailure, TrajectoryResult, reference_types

__all__ = ["DeviceProblem", "RunOutput", "run_gpu", "run_sharded", "partition_trajectories",
           "raise_for_status", "stats_dict", "flops_model", "autotune_variant",
           "candidate_variants", "run_logged", "shard_range", "combine_blocks"]


def partition_trajectories(n_total: int, n_workers: int) -> list[int]:
    """Counts per worker: sum n_total, max - min <= 1, remainder to the
    lowest ranks (cluster.py:369-377)."""
    if n_total < 1:
        raise ValueError("n_total must be positive")
    if n_workers < 1:
        raise ValueError("n_workers must be positive")
    base, rem = divmod(n_total, n_workers)
    return [base + 1 if r < rem else base for r in range(n_workers)]


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Rank ``rank``'s contiguous share of the global trajectory indices:
    whole reduction blocks of ``native.BLOCK`` trajectories, the blocks
    split by the reference's partition rule (cluster.py:369-377, counts
    differing by at most one block).  Block-aligned shards make the
    multi-GPU ensemble sums bitwise equal to a single run's (run_sharded)."""
    n_blocks = -(-n_total // native.BLOCK)
    counts = partition_trajectories(n_blocks, world) if n_blocks >= world else \
        [1 if r < n_blocks else 0 for r in range(world)]
    b0 = sum(counts[:rank])
    return min(b0 * native.BLOCK, n_total), min((b0 + counts[rank]) * native.BLOCK, n_total)


def combine_blocks(block_sum: np.ndarray, block_sumsq: np.ndarray):
    """Stage 2 of the fixed-order ensemble reduction on the host, in the
    order of the device's ensemble_final (qtm_capi.cu): ((0 + b_0) + b_1) + ..."""
    s = np.zeros(block_sum.shape[1:])
    s2 = np.zeros(block_sum.shape[1:])
    for b in range(block_sum.shape[0]):
        s = s + block_sum[b]
        s2 = s2 + block_sumsq[b]
    return s, s2


def _inside(istate: int, detail: str, problem=None) -> OdeFailure:
    # run_single_trajectory re-raises solver failures with this suffix
    # (trajectory.py:247-248)
    failure = reference_types(problem)[0]
    inner = failure(istate, detail)
    return failure(istate, f"{inner} (inside trajectory)")


def raise_for_status(code: int, err: dict, problem=None) -> None:
    """Raise the reference's exception for a failing trajectory: an
    ``OdeFailure`` that is also ``mcwf.ode.OdeFailure`` when the caller uses
    the reference package (problem.reference_types), else ValueError /
    RuntimeError exactly where the reference raises them."""
    t, h = err.get("t", 0.0), err.get("h", 0.0)
    if code == native.ERR_MAX_STEPS:
        raise _inside(-1, f"max_steps = {err.get('max_steps')} exhausted in trajectory segment "
                          f"at t = {t:g}", problem)
    if code == native.ERR_REPEATED_ERRTEST:
        raise _inside(-4, f"repeated error-test failures at t = {t:g}", problem)
    if code == native.ERR_STEP_COLLAPSE:
        raise _inside(-5, f"step size collapsed to {h:g} at t = {t:g}", problem)
    if code == native.ERR_CORRECTOR:
        raise _inside(-5, f"corrector failed to converge at t = {t:g}", problem)
    if code == native.ERR_BRACKET:
        f_lo, f_hi, r = err.get("aux", (0.0, 0.0, 0.0))
        raise RuntimeError(f"jump bracket violated: norm_sq({t:g}) = {f_lo:g}, "
                           f"norm_sq({h:g}) = {f_hi:g}, r = {r:g}")
    if code == native.ERR_NO_SUPPORT:
        raise ValueError("no collapse channel has support on the state")
    if code == native.ERR_ZERO_VECTOR:
        raise ValueError("expectation of a zero vector")
    raise RuntimeError(f"trajectory engine error {code}")


def stats_dict(row) -> dict:
    return {name: int(row[i]) for i, name in enumerate(native.STAT_NAMES)}


def flops_model(stats_total: dict, packed: PackedProblem) -> float:
    """Algorithmic FP64 flops of all step attempts:
    per attempt m (8 nnz + 15 d) + d (q(q+1) + 4(q+1) + 13).

    BDF (modified Newton, ode.py:379-423): per Newton iteration the SpMV
    (8 nnz), the two triangular solves (8 d^2) and the residual / update /
    WRMS (16 d); per attempt the predict, error test and commit; per LU
    factorisation of I - h l0 G 8/3 d^3 (complex rank-1 updates) + 2 nnz."""
    d, nnz = packed.dim, packed.g.nnz
    m = stats_total["corr_iters"]
    att = stats_total["attempts"]
    if getattr(packed, "method", 0) == 1:
        return float(m * (8 * nnz + 8 * d * d + 16 * d)
                     + d * (stats_total["sum_qq1"] + 4 * (stats_total["sum_q"] + att) + 8 * att)
                     + stats_total.get("lu_factor", 0) * (8.0 / 3.0 * d ** 3 + 2 * nnz))
    return float(m * (8 * nnz + 15 * d)
                 + d * (stats_total["sum_qq1"] + 4 * (stats_total["sum_q"] + att) + 13 * att))


def bytes_model(stats_total: dict, packed: PackedProblem) -> float:
    """HBM bytes the state-streaming design would move:
    16 d (2 (q+1) + 2) per attempt."""
    d = packed.dim
    att = stats_total["attempts"]
    return float(16 * d * (2 * (stats_total["sum_q"] + att) + 2 * att))


def spmv_value_bytes(packed: PackedProblem, shape=None) -> int:
    """Dictionary-value bytes one staged SpMV loads per thread-row set (summed
    over G's stored entries).  16 per entry in general.  On the wide variants
    (several rows per thread, pipelined SpMV; `sell_uses_dom` in
    csrc/qtm_traj.cuh, rule restated from `build_sell` in csrc/qtm_capi.cu)
    the entries of a dominant purely imaginary value (at least half of the
    entries) load nothing, and the other purely imaginary values (if at least
    a quarter of the entries) load 8 bytes."""
    nnz = packed.g.nnz
    wide = (shape is not None and shape[1] > 1 and shape[2] > 0 and not packed.td
            and os.environ.get("QTM_DOM", "7") != "0")
    if not wide or nnz == 0:
        return 16 * nnz
    mode = int(os.environ.get("QTM_DOM", "7"))
    vals = np.asarray(packed.g.values).view(np.float64).reshape(-1, 2)
    imag = vals[:, 0].view(np.uint64) == 0  # re is +0.0 bit for bit
    n_dom = 0
    if imag.any():
        _, counts = np.unique(vals[imag, 1].view(np.uint64), return_counts=True)
        best = int(counts.max())
        if (mode & 1) and 2 * best >= nnz:
            n_dom = best
    n_other = int(imag.sum()) - n_dom
    if not (mode & 2) or 4 * n_other < nnz:
        n_other = 0
    return 16 * (nnz - n_dom - n_other) + 8 * n_other


def smem_model(stats_total: dict, packed: PackedProblem, shape=None) -> float:
    """Shared-memory bytes the Adams trajectory kernel moves by construction
    (DESIGN.md §3): per corrector iteration the staged-operator SpMV reads an
    entry word and a 16-byte gathered x per nonzero (20 nnz) plus the
    dictionary values (`spmv_value_bytes`: 16 per nonzero in general, fewer
    on the wide variants when G's off-diagonals are purely imaginary), and
    the update reads the iterate and the weight and writes the next iterate
    (40 d); per attempt the predicted z0 is published once (16 d).
    Reductions, row 0 of the TMEM variant and recording come on top, so the
    measured wavefronts (ncu) are higher.  `shape` = the kernel variant's
    (threads, components, register rows)."""
    d, nnz = packed.dim, packed.g.nnz
    per_spmv = 20 * nnz + spmv_value_bytes(packed, shape)
    return float(stats_total["corr_iters"] * (per_spmv + 40 * d) + stats_total["attempts"] * 16 * d)


@dataclass
class RunOutput:
    sum: np.ndarray
    sumsq: np.ndarray
    values: np.ndarray | None
    stats: np.ndarray | None
    stats_total: np.ndarray
    status: np.ndarray | None
    jump_count: np.ndarray | None
    jump_t: np.ndarray | None
    jump_idx: np.ndarray | None
    error: dict | None
    rc: int
    kernel_ms: float
    total_ms: float
    variant: int
    grid: int
    launches: int
    count: int
    n_failed: int = 0
    psi: np.ndarray | None = None  # [count, n_psi_points, dim] complex, psi_points only
    block_sum: np.ndarray | None = None    # [n_blocks, n_expect, n_pts] (block_sums=True)
    block_sumsq: np.ndarray | None = None


def _p(a, t=C.POINTER(C.c_double)):
    return a.ctypes.data_as(t) if a is not None else None


class DeviceProblem:
    """A problem resident in one GPU's HBM (qtm_problem handle)."""

    def __init__(self, problem, *, device: int = 0, variant: int = -1,
                 h0_first: float | None = None):
        self.packed = problem if isinstance(problem, PackedProblem) else \
            pack_problem(problem, h0_first=h0_first)
        self.device = device
        L = native.lib()
        pk = self.packed
        keep = []

        def csr(m):
            keep.extend([m.row_ptr, m.col_ind, m.values])
            return native.QtmCsr(_p(m.row_ptr, C.POINTER(C.c_int64)),
                                 _p(m.col_ind, C.POINTER(C.c_int64)), _p(m.values), m.nnz)

        coll = (native.QtmCsr * max(1, pk.n_collapse))(*[csr(c) for c in pk.collapse])
        expt = (native.QtmCsr * max(1, pk.n_expect))(*[csr(e) for e in pk.expect])
        tds = (native.QtmCsr * max(1, pk.n_td))(*[csr(m) for m in pk.td])
        desc = native.QtmProblemDesc(
            native.ABI_VERSION, pk.dim, csr(pk.g), pk.n_collapse, coll, pk.n_expect, expt,
            _p(pk.psi0), pk.t_from, pk.t_to, pk.n_steps, _p(pk.times), pk.method, pk.rtol, pk.atol,
            pk.max_order, pk.max_steps, pk.h0_first, _p(pk.l_table), _p(pk.tau1), _p(pk.tau2),
            _p(pk.tau3), device, variant, pk.n_td, tds, _p(pk.td_coef))
        handle = C.c_void_p()
        rc = L.qtm_problem_create(C.byref(desc), C.byref(handle))
        if rc != 0:
            raise RuntimeError(f"qtm_problem_create failed ({rc}): {native.last_error()}")
        self._handle = handle
        self._lock = threading.Lock()

    def max_resident(self) -> int:
        """Trajectories in flight at once (persistent grid size)."""
        out = C.c_int32()
        if native.lib().qtm_max_resident(self._handle, C.byref(out)) != 0:
            raise RuntimeError(native.last_error())
        return out.value

    def layout(self) -> dict:
        """Nordsieck history placement: register rows, shared-memory rows
        (the rest in global scratch) and dynamic shared memory per CTA."""
        r, s, b = C.c_int32(), C.c_int32(), C.c_int64()
        if native.lib().qtm_problem_layout(self._handle, C.byref(r), C.byref(s), C.byref(b)) != 0:
            raise RuntimeError(native.last_error())
        v = native.lib().qtm_problem_variant(self._handle)
        return {"reg_rows": r.value, "smem_rows": s.value, "smem_bytes": b.value,
                "tmem_rows": native.variant_tmem_rows(v) if v >= 0 else 0, "variant": v}

    def close(self):
        if getattr(self, "_handle", None):
            native.lib().qtm_problem_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def run(self, seed: int, traj_begin: int, traj_end: int, *, stream: str = "philox",
            script=None, script_fallback: float = 0.999999, max_jumps: int = 0,
            per_trajectory: bool = True, resident: bool = False,
            cuda_stream: int | None = None, psi_points=None,
            block_sums: bool = False) -> RunOutput:
        """Integrate global trajectories [traj_begin, traj_end).  With
        ``per_trajectory`` the per-trajectory series, counters and jump logs
        come back too; ``resident`` skips those copies entirely.
        ``psi_points`` (grid indices) returns each trajectory's state at
        those points -- the interpolated, unnormalised psi the reference
        passes to record_expectation (trajectory.py:206-214)."""
        if self._handle is None:
            raise RuntimeError("device problem already closed")
        pk = self.packed
        n = traj_end - traj_begin
        n_out = pk.n_expect * pk.n_pts
        script_arr = script_len = None
        stride = 0
        if stream == "scripted":
            rows = [list(map(float, s)) for s in script]
            if len(rows) != n:
                raise ValueError("scripted stream needs one script row per trajectory")
            stride = max(1, max((len(r) for r in rows), default=1))
            script_arr = np.zeros((n, stride))
            script_len = np.zeros(n, np.int64)
            for i, r in enumerate(rows):
                script_arr[i, : len(r)] = r
                script_len[i] = len(r)
        pts = None if psi_points is None else np.ascontiguousarray(psi_points, dtype=np.int64)
        args = native.QtmRunArgs(int(seed) & 0xFFFFFFFFFFFFFFFF, traj_begin, traj_end,
                                 native.STREAM_KINDS[stream], _p(script_arr),
                                 _p(script_len, C.POINTER(C.c_int64)), stride, script_fallback,
                                 max_jumps, cuda_stream, 0 if pts is None else len(pts),
                                 _p(pts, C.POINTER(C.c_int64)))
        psi = None if pts is None else np.zeros((n, len(pts), pk.dim), dtype=np.complex128)
        s = np.zeros(max(n_out, 1))
        s2 = np.zeros(max(n_out, 1))
        tot = np.zeros(native.NSTATS, np.int64)
        want = per_trajectory and not resident
        vals = np.zeros((n, pk.n_expect, pk.n_pts)) if want else None
        stats = np.zeros((n, native.NSTATS), np.int64) if want else None
        status = np.zeros(n, np.int32) if want else None
        jc = np.zeros(n, np.int64) if want else None
        jt = np.zeros((n, max_jumps)) if want and max_jumps else None
        ji = np.zeros((n, max_jumps), np.int32) if want and max_jumps else None
        out = native.QtmRunOut(_p(s), _p(s2), _p(vals), _p(stats, C.POINTER(C.c_int64)),
                               _p(tot, C.POINTER(C.c_int64)), _p(status, C.POINTER(C.c_int32)),
                               _p(jc, C.POINTER(C.c_int64)), _p(jt),
                               _p(ji, C.POINTER(C.c_int32)))
        if psi is not None:
            out.psi = psi.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))
        bs = bs2 = None
        if block_sums:
            nb = -(-n // native.BLOCK)
            bs = np.zeros((nb, pk.n_expect, pk.n_pts))
            bs2 = np.zeros((nb, pk.n_expect, pk.n_pts))
            if n_out > 0 and n > 0:
                out.block_sum = _p(bs)
                out.block_sumsq = _p(bs2)
        L = native.lib()
        with self._lock:
            fn = L.qtm_run_resident if resident else L.qtm_run
            rc = fn(self._handle, C.byref(args), C.byref(out))
        err = None
        if rc != 0:
            if rc in (native.ERR_ARGS, native.ERR_CUDA, native.ERR_UNSUPPORTED):
                raise RuntimeError(f"qtm_run failed ({rc}): {native.last_error()}")
            e = out.error
            err = {"code": e.code, "traj": e.traj, "t": e.t, "h": e.h, "max_steps": e.max_steps,
                   "aux": (e.aux0, e.aux1, e.aux2)}
        return RunOutput(s[:n_out].reshape(pk.n_expect, pk.n_pts),
                         s2[:n_out].reshape(pk.n_expect, pk.n_pts), vals, stats, tot, status, jc,
                         jt, ji, err, rc, out.kernel_ms, out.total_ms, out.variant, out.grid,
                         out.launches, n, int(out.n_failed), psi, bs, bs2)


_TUNED: dict = {}


def candidate_variants(dim: int, time_dependent: bool = False) -> list[int]:
    """Kernel variants able to hold a state of this dimension without
    wasting more than half of their lanes (the smallest fit always counts),
    among those built with / without the time-dependent terms."""
    vs = native.variants()
    small = [i for i in range(len(vs)) if 0 < native.variant_small(i)[0]]
    fits = [i for i, (t, e, _) in enumerate(vs)
            if i not in small and t * e >= dim
            and native.variant_time_dependent(i) == time_dependent]
    cands = []
    if fits:
        smallest = min(vs[i][0] * vs[i][1] for i in fits)
        cands = [i for i in fits if vs[i][0] * vs[i][1] <= max(2 * dim, smallest)]
    # one thread per trajectory (constant generators only): the smallest d_max >= dim
    dms = [native.variant_small(i)[0] for i in small if native.variant_small(i)[0] >= dim]
    if dms and not time_dependent:
        cands += [i for i in small if native.variant_small(i)[0] == min(dms)]
    return cands


def autotune_variant(packed: PackedProblem, *, device: int = 0, sample: int | None = None,
                     seed: int = 987654321, n_total: int | None = None) -> int:
    """Pick the fastest kernel variant for this problem by timing each
    candidate on a sample of trajectories (result cached per problem digest,
    device and run size).  The register budget for the Nordsieck history is
    the main trade-off: enough rows for the orders the problem actually
    reaches, but no more than needed to keep more warps resident.  With
    ``n_total`` the sample never exceeds the run: a run that fits in one
    wave is latency-bound (c1: 500 trajectories), where the variant with the
    shortest per-trajectory chain wins rather than the one with most CTAs."""
    key = (packed.digest, device, n_total)
    if key in _TUNED:
        return _TUNED[key]
    cands = candidate_variants(packed.dim, packed.n_td > 0)
    if len(cands) <= 1:
        _TUNED[key] = cands[0] if cands else -1
        return _TUNED[key]
    def timed(v, reps):
        with DeviceProblem(packed, device=device, variant=v) as dp:
            # enough trajectories for several waves of this variant's
            # persistent grid, so the comparison is not decided by the tail
            n = sample or min(max(6 * dp.max_resident(), 1024), 8192, n_total or 8192)
            return min(dp.run(seed, 0, n, resident=True).kernel_ms for _ in range(reps)) / n

    # one pass over every candidate, then the three fastest again (best of
    # two), so run-to-run noise of a few percent does not pick the runner-up
    first = sorted((timed(v, 1), v) for v in cands)
    best_ms, best = min((min(ms, timed(v, 2)), v) for ms, v in first[:3])
    _TUNED[key] = best
    return best


def _result(pk: PackedProblem, out: RunOutput, n_ok: int, jumps, problem=None) -> TrajectoryResult:
    stats = stats_dict(out.stats_total)
    stats["failed"] = out.n_failed
    return reference_types(problem)[1](pk.times, out.sum / max(n_ok, 1), n_ok, jumps, sumsq=out.sumsq,
                            stats=stats)


def _jump_list(out: RunOutput):
    if out.jump_t is None or int(out.jump_count.max(initial=0)) > out.jump_t.shape[1]:
        raise RuntimeError("jump log truncated: run with a larger max_jumps "
                           "(run_logged grows it automatically)")
    jumps = []
    for i in range(out.count):
        for j in range(int(out.jump_count[i])):
            jumps.append((float(out.jump_t[i, j]), int(out.jump_idx[i, j])))
    return jumps


def run_logged(dp: "DeviceProblem", seed: int, begin: int, end: int, *, max_jumps: int = 1024,
               **kw) -> RunOutput:
    """``dp.run`` with a complete jump log, as the reference keeps every jump
    (trajectory.py:238-239): the device logs the first ``max_jumps`` jumps of
    each trajectory and counts all of them; if any trajectory jumped more
    often, the (deterministic) run is repeated with the capacity raised to
    the largest count."""
    out = dp.run(seed, begin, end, max_jumps=max(1, max_jumps), per_trajectory=True, **kw)
    most = int(out.jump_count.max(initial=0))
    if most > out.jump_t.shape[1]:
        out = dp.run(seed, begin, end, max_jumps=most, per_trajectory=True, **kw)
    return out


def run_gpu(problem, n_total: int, master_seed: int, *, device: int = 0,
            stream: str = "philox", log_jumps: bool | None = None, max_jumps: int = 1024,
            variant: int = -1, on_failure: str = "raise") -> TrajectoryResult:
    """Drop-in for ``mcwf.run_inline(problem, n_total, master_seed)``:
    trajectories 0..n_total-1 on one GPU, count-weighted mean over them.

    ``on_failure="raise"`` (default) raises the reference's exception for
    the lowest failing trajectory, as run_inline would; ``"exclude"``
    averages over the trajectories that completed and reports the failures
    in ``result.stats["failed"]``."""
    if n_total < 1:
        raise ValueError("n_total must be positive")
    if on_failure not in ("raise", "exclude"):
        raise ValueError("on_failure must be 'raise' or 'exclude'")
    with DeviceProblem(problem, device=device, variant=variant) as dp:
        if log_jumps is None:
            log_jumps = dp.packed.log_jumps
        if log_jumps:
            out = run_logged(dp, master_seed, 0, n_total, stream=stream, max_jumps=max_jumps)
        else:
            out = dp.run(master_seed, 0, n_total, stream=stream, per_trajectory=False)
        if out.rc != 0 and on_failure == "raise":
            raise_for_status(out.rc, out.error, problem)
        return _result(dp.packed, out, n_total - out.n_failed,
                       _jump_list(out) if log_jumps else None, problem)


def run_sharded(problem, n_total: int, master_seed: int, *, rank: int, world_size: int,
                stream: str = "philox", device: int | None = None, runner=None,
                group=None, on_failure: str = "raise", variant: int = -1) -> TrajectoryResult | None:
    """One rank of a multi-GPU run (one process per GPU, torch.distributed
    initialised by the caller).  Rank r integrates its contiguous,
    block-aligned range of global trajectory indices (shard_range); the
    reduction-block partials, counters, failure count and every rank's first
    failing trajectory travel in ONE float64 SUM all-reduce:

        [block_sum | block_sumsq | stats | n_failed | first_fail[world] | setup_error[world]]

    Every slot is written by exactly one rank (the others contribute 0), so
    the all-reduce is exact, and every rank then adds the blocks in block
    order like the device's own ensemble_final: the sums are bitwise those of
    a single-GPU run, whatever the number of ranks.  (first_fail[r] = 1 + the
    global index of rank r's lowest failing trajectory, 0 if none.)  A rank
    whose device setup or launch raises still joins the collective with
    setup_error[r] = 1, so no rank is left waiting, and every rank raises
    afterwards.  Returns the TrajectoryResult on every rank.

    ``runner(packed, seed, begin, end, stream) -> RunOutput`` (with
    block_sum / block_sumsq) defaults to the device engine on ``device``
    (= rank); the CPU multi-process tests inject the oracle here to check
    the sharding and reduction logic with gloo."""
    import torch
    import torch.distributed as dist

    packed = problem if isinstance(problem, PackedProblem) else pack_problem(problem)
    begin, end = shard_range(n_total, world_size, rank)
    n_out = packed.n_expect * packed.n_pts
    n_blocks = -(-n_total // native.BLOCK)
    out, local_exc = None, None
    try:
        if end <= begin:
            out = None
        elif runner is None:
            dev = rank if device is None else device
            with DeviceProblem(packed, device=dev, variant=variant) as dp:
                out = dp.run(master_seed, begin, end, stream=stream, per_trajectory=False,
                             resident=True, block_sums=True)
        else:
            out = runner(packed, master_seed, begin, end, stream)
    except Exception as exc:  # joined below, re-raised after the collective
        local_exc = exc
    tab = 2 * n_blocks * n_out
    base = tab + native.NSTATS + 1
    vec = np.zeros(base + 2 * world_size)
    if local_exc is not None:
        vec[base + world_size + rank] = 1
    elif out is not None:
        b0 = begin // native.BLOCK
        nb = out.block_sum.shape[0]
        blocks = vec[:tab].reshape(2, n_blocks, n_out)
        blocks[0, b0:b0 + nb] = out.block_sum.reshape(nb, n_out)
        blocks[1, b0:b0 + nb] = out.block_sumsq.reshape(nb, n_out)
        vec[tab:tab + native.NSTATS] = out.stats_total
        vec[tab + native.NSTATS] = out.n_failed
        if out.rc != 0:
            vec[base + rank] = 1 + int(out.error["traj"])
    backend = dist.get_backend(group)
    tdev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else \
        torch.device("cpu")
    buf = torch.from_numpy(vec).to(tdev)
    dist.all_reduce(buf, group=group)
    host = buf.cpu().numpy()
    if local_exc is not None:
        raise local_exc
    bad = [r for r in range(world_size) if host[base + world_size + r] != 0]
    if bad:
        raise RuntimeError(f"rank(s) {bad} failed before integrating their trajectories")
    fails = [int(x) - 1 for x in host[base:base + world_size] if x != 0]
    if fails and on_failure == "raise":
        first_fail = min(fails)
        if out is not None and out.rc != 0 and out.error["traj"] == first_fail:
            raise_for_status(out.rc, out.error, problem)
        raise RuntimeError(f"trajectory {first_fail} failed on another rank")
    blocks = host[:tab].reshape(2, n_blocks, packed.n_expect, packed.n_pts)
    s, s2 = combine_blocks(blocks[0], blocks[1])
    stats = stats_dict(host[tab:tab + native.NSTATS].astype(np.int64))
    stats["failed"] = int(host[tab + native.NSTATS])
    n_ok = n_total - stats["failed"]
    return reference_types(problem)[1](packed.times, s / max(n_ok, 1), n_ok, None, sumsq=s2,
                                       stats=stats)
