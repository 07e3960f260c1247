"""Benchmark: trajectories/sec of the ensemble run on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

A "step" integrates the whole trajectory ensemble of the configuration
(default c4: dissipative transverse-field Ising chain, d=1024, 4096
trajectories -- the config BASELINE.json quotes at 1/2/4/8 B200) and
reduces <sigma_z^i>(t) over it.  N>1 runs one process per GPU under
torchrun; the trajectory range is sharded contiguously (strong scaling:
the 4096 trajectories are split over the ranks) and the per-point sums
are combined with one NCCL all-reduce inside the e2e leg.

Timing: W untimed steps, then K steps between a barrier +
torch.cuda.synchronize() on both sides, CUDA events on the launching stream
(the library launches on torch's current stream), max over ranks.  A
256 MiB buffer (> 126 MB L2) is overwritten between timed steps.

`--impl reference` times the reference's CPU path -- the C restatement in
oracle/ (the reference is Python+numba; nothing of it travels to the GPU
box) -- on all host cores for a bounded trajectory sample per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

SEED = 987654321
WORKLOADS = {
    "c1": "c1: driven damped two-level atom (d=2), 500 trajectories, 201 output times",
    "c2": "c2: driven damped cavity (d=20), 5000 trajectories, 301 output times",
    "c3": "c3: Jaynes-Cummings cavity+qubit (d=80), 20000 trajectories, 501 output times",
    "c4": "c4: dissipative transverse-field Ising L=10 (d=1024, CSR 11 nnz/row), "
          "4096 trajectories, 101 output times",
    "c5": "c5: two coupled lossy Kerr cavities (d=900, CSR), 100000 trajectories, 401 output times",
    "c4td": "c4td: c4 with a modulated transverse field h(t) = 0.7 + 0.3 cos(2t) "
            "(time-dependent H, d=1024), 4096 trajectories, 101 output times",
}
METRIC = "trajectories/sec (ensemble <O>(t))"


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region.

    NVML is polled from a background thread (every 250 ms) instead of an
    nvidia-smi subprocess: the subprocess's own queries were measured to stall
    the GPU work of this process by ~100 ms per sample on the B200 pool.
    QTM_CLOCKS=smi selects the nvidia-smi sampler, QTM_CLOCKS=off disables."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device: int, interval: float = 0.25):
        self.device = device
        self.interval = interval
        self.mode = os.environ.get("QTM_CLOCKS", "nvml")
        self.samples = []
        self._stop = None
        self._thread = None
        self.proc = None
        self.path = None

    def start(self):
        if self.mode == "off":
            return
        if self.mode == "smi":
            return self._start_smi()
        try:
            import threading
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
        except Exception:
            return self._start_smi()
        self._stop = threading.Event()

        def loop():
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, smax, rs))
                except Exception:
                    pass
                self._stop.wait(self.interval)

        self._thread = threading.Thread(target=loop, daemon=True)
        self._thread.start()

    def _start_smi(self):
        query = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={query}",
                 "--format=csv,noheader,nounits", "-lms", "200", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=5)
            if not self.samples:
                return None
            names = [n for n, bit in self.REASONS.items()
                     if any(rs & bit for _, _, rs in self.samples)]
            return {"sm_mhz": statistics.median(s for s, _, _ in self.samples),
                    "sm_max_mhz": max(m for _, m, _ in self.samples), "reasons": sorted(names),
                    "samples": len(self.samples), "source": "nvml"}
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        finally:
            os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(rows), "source": "nvidia-smi"}


def cpu_reference(packed, sample: int, steps: int, warmup: int, threads: int):
    """The reference CPU path (oracle port, all host threads) on a bounded
    sample of trajectories per step."""
    from oracle import oracle
    oracle.build()
    for _ in range(warmup):
        oracle.run(packed, SEED, 0, sample, n_threads=threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        r = oracle.run(packed, SEED, 0, sample, n_threads=threads)
        times.append(time.perf_counter() - t0)
        if r["rc"] not in (0, -1, -4, -5, -6):
            raise RuntimeError(f"oracle failed: {r['error']}")
        done = sample - int(np.count_nonzero(r["status"]))
    return done / (sum(times) / len(times)), sum(times) / len(times)


CPU_SAMPLE_PER_THREAD = {"c1": 128, "c2": 32, "c3": 16, "c4": 8, "c5": 1, "c4td": 8}


def profiled_traffic(config: str):
    """DRAM bytes per launch of the trajectory kernel from the newest committed
    ncu --set full capture of this config
    (profiles/r*_<config>_traj_kernel_raw_selected.csv), or None."""
    import glob
    # round-1 captures are r0<N>_*, round 2's r2_*: the last name is the newest
    found = sorted(glob.glob(os.path.join(REPO, "profiles", f"r*_{config}_traj_kernel_raw_selected.csv")))
    if not found:
        return None
    path = found[-1]
    vals = {}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    with open(path) as f:
        for line in f:
            parts = line.strip().split(",")
            if len(parts) == 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                vals[parts[0]] = float(parts[2]) * scale.get(parts[1], 1.0)
    if len(vals) != 2:
        return None
    return {"bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
            "source": os.path.relpath(path, REPO)}


def profiled_smem_pct(config: str):
    """Shared-memory data-pipe utilisation of the trajectory kernel (per cent of
    peak, sustained over the launch) from the newest committed ncu capture."""
    import glob
    found = sorted(glob.glob(os.path.join(REPO, "profiles", f"r*_{config}_traj_kernel_raw_selected.csv")))
    for path in reversed(found):
        with open(path) as f:
            for line in f:
                parts = line.strip().split(",")
                if len(parts) == 3 and parts[0] == \
                        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed":
                    return {"pct": float(parts[2]), "source": os.path.relpath(path, REPO)}
    return None


def _sum_over_ranks(dist, torch, local, x, world):
    if world == 1:
        return x
    dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return float(t.item())


def build_problem(args):
    """The config's problem; ``--method bdf`` swaps in the BDF family (same
    tolerances) -- the reference's general engine, ode.py:334-423."""
    import dataclasses

    from paper_1810_03047_b200 import configs
    from paper_1810_03047_b200.problem import OdeConfig
    p = configs.build(args.config)
    if args.method != "adams":
        p = dataclasses.replace(p, ode=OdeConfig(method=args.method, rtol=p.ode.rtol,
                                                 atol=p.ode.atol))
    return p


REF_ENGINE_SAMPLE = {"c1": 2000, "c2": 160, "c3": 96, "c4": 128, "c5": 16, "c4td": 64}


def reference_engine(config: str, workers: int):
    """The reference's OWN CPU engine (Python + numba, pip-installed into
    baseline/_ref) timed on this host: ``mcwf.run_local_farm`` (cluster.py:493)
    over a bounded sample of the config, problem built by the reference's
    constructors (tests/golden/ref_configs.py), numba compiled in the parent
    before the fork (untimed).  None when the reference package is absent."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mcwf")) or config not in REF_ENGINE_SAMPLE \
            or config == "c4td":
        return None
    sys.path.insert(0, os.path.join(REPO, "tests", "golden"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "qtm_numba"))
    try:
        import ref_configs  # noqa: F401  (puts baseline/_ref on sys.path)
        import mcwf
        from oracle.streams import PhiloxStream
    except ImportError:
        return None
    problem = ref_configs.CONFIGS[config](log_jumps=False)
    mcwf.run_single_trajectory(problem, PhiloxStream(SEED, 0))  # numba JIT, untimed
    n = REF_ENGINE_SAMPLE[config]
    t0 = time.perf_counter()
    mcwf.run_local_farm(problem, n, workers, SEED)
    sec = time.perf_counter() - t0
    return {"value": n / sec, "unit": "trajectories/s", "cores": workers, "kind": "reference",
            "sample": f"{n} trajectories of {config}: mcwf.run_local_farm(problem, {n}, {workers}, "
                      f"{SEED}) from baseline/_ref (the reference's own Python + numba engine, "
                      f"one worker process per host thread)"}


def run_reference_arm(args, rank, world):
    from paper_1810_03047_b200.packing import pack_problem
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    packed = pack_problem(build_problem(args))
    sample = CPU_SAMPLE_PER_THREAD[args.config] * threads
    value, sec = cpu_reference(packed, sample, args.steps, args.warmup, threads)
    desc = (f"{sample} trajectories of {args.config} per step (global indices 0..{sample - 1}, "
            f"Philox streams), oracle/mcwf_oracle.c on {threads} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "trajectories/s",
            "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "config": args.config,
                       "method": args.method, "trajectories_per_step": sample},
            "cpu_baseline": {"value": value, "unit": "trajectories/s", "cores": threads,
                             "kind": "port", "sample": desc},
            "e2e": {"value": value, "unit": "trajectories/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if args.method == "adams":
        try:
            line["reference_engine"] = reference_engine(args.config, threads)
        except Exception as exc:  # the port's line stands on its own
            line["reference_engine"] = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(cmd: list, n: int, env: dict | None = None) -> int:
    """Start ``cmd`` as ``n`` ranks of one job, the way torchrun would (one
    process per GPU; RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* in the
    environment, rendezvous on 127.0.0.1) -- bench.py's own launcher for
    ``--gpus N`` outside torchrun, as the reference farm spawns its own
    workers (cluster.py:493-507).  Rank 0's stdout is this process's stdout;
    the other ranks' stdout goes to stderr.  Returns the worst exit code."""
    base = dict(os.environ if env is None else env)
    base.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE=str(n),
                LOCAL_WORLD_SIZE=str(n))
    base.setdefault("NCCL_DEBUG", "INFO")
    procs = []
    for r in range(n):
        e = dict(base, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen(cmd, env=e, stdout=None if r == 0 else sys.stderr))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--variant", type=int, default=-2,
                    help="kernel variant (-1: by dimension, -2: autotune during warm-up)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline leg")
    ap.add_argument("--method", default="adams", choices=["adams", "bdf"],
                    help="ODE method family (bdf: modified Newton with a dense LU per trajectory)")
    ap.add_argument("--trajectories", type=int, default=0,
                    help="override the config's trajectory count (exploration only)")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # not under torchrun: start the N ranks ourselves
        sys.exit(launch_ranks([sys.executable, os.path.abspath(__file__)] +
                              list(sys.argv[1:] if argv is None else argv), args.gpus))
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")

    import torch
    import torch.distributed as dist

    from paper_1810_03047_b200 import configs, native
    from paper_1810_03047_b200.configs import N_TRAJECTORIES
    from paper_1810_03047_b200.engine import (smem_model, spmv_value_bytes, DeviceProblem, autotune_variant, bytes_model,
                                              flops_model, run_sharded, shard_range, stats_dict)
    from paper_1810_03047_b200.packing import pack_problem

    n_dev = torch.cuda.device_count()
    if local >= n_dev:  # more ranks than GPUs (functional test of the multi-rank path only)
        local = local % n_dev
    torch.cuda.set_device(local)
    if world > 1:
        if n_dev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            # NCCL refuses two ranks on one GPU; the tiny end-of-run reduction
            # then goes through gloo (never the case on an 8-GPU box)
            dist.init_process_group("gloo")
    stream = torch.cuda.current_stream(local)
    problem = build_problem(args)
    packed = pack_problem(problem)
    n_total = (args.trajectories or N_TRAJECTORIES[args.config]) * \
        (world if args.scaling == "weak" else 1)
    begin, end = shard_range(n_total, world, rank)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # the clock sampler starts before the warm-up so that nvidia-smi's own
    # start-up is over before the timed region
    clocks = ClockSampler(local)
    clocks.start()
    if args.method == "bdf":
        args.variant = -1  # one BDF kernel per block size (qtm_bdf.cuh)
    if args.variant == -2:  # untimed: choose the kernel variant on a sample (rank 0's
        # choice everywhere, so every rank runs the same kernel)
        if rank == 0:
            args.variant = autotune_variant(packed, device=local, n_total=end - begin)
        if world > 1:
            dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
            v = torch.tensor([args.variant], dtype=torch.int64, device=dev)
            dist.broadcast(v, src=0)
            args.variant = int(v.item())
    dp = DeviceProblem(packed, device=local, variant=args.variant)
    for _ in range(args.warmup):
        flush.zero_()  # also loads the fill kernel's module before timing (lazy loading)
        out = dp.run(SEED, begin, end, resident=True, cuda_stream=stream.cuda_stream)
        if out.rc not in (0, -1, -4, -5, -6):  # trajectory failures are the reference's own
            raise RuntimeError(f"warm-up run failed: {out.error}")

    # ---- device-timed leg: inputs resident in HBM -------------------------
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    kernel_ms = []
    launches = 0
    outs = []
    step_ev = []
    for _ in range(args.steps):
        flush.zero_()
        e_a = torch.cuda.Event(enable_timing=True)
        e_a.record(stream)
        out = dp.run(SEED, begin, end, resident=True, cuda_stream=stream.cuda_stream)
        kernel_ms.append(out.kernel_ms)
        launches += out.launches
        outs.append(out)
        step_ev.append(e_a)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    step_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    per_step = [step_ev[i].elapsed_time(step_ev[i + 1] if i + 1 < len(step_ev) else ev1)
                for i in range(len(step_ev))]
    n_failed = int(_sum_over_ranks(dist, torch, local, outs[-1].n_failed, world))
    # completed trajectories per second (a trajectory on which the reference
    # controller itself collapses -- OdeFailure -5 -- is excluded)
    value = (n_total - n_failed) / (step_ms * 1e-3)

    # roofline of the trajectory kernel (dominant: >99 % of the step)
    st = stats_dict(outs[-1].stats_total)
    k_ms = float(np.mean(kernel_ms))
    flops = flops_model(st, packed)
    peak = native.fp64_peak_tflops(local)
    dmma_peak = native.dmma_peak_tflops(local)
    achieved = flops / (k_ms * 1e-3) / 1e12
    hbm_equiv = bytes_model(st, packed) / (k_ms * 1e-3) / 1e9
    hbm_peak = None
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            hbm_peak = float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        hbm_peak = 6650.0  # B200_PROFILING.md fallback ("of fallback")
    layout = dp.layout()
    dp.close()
    # shared-memory side of the same kernel: model bytes / kernel time against
    # 128 B per clock per SM at the clock measured under load
    smem = None
    if args.method == "adams" and not native.variant_small(outs[-1].variant)[0]:
        n_sm = torch.cuda.get_device_properties(local).multi_processor_count
        mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz") or 1965
        smem_peak = 128.0 * n_sm * mhz * 1e6 / 1e12
        shape = native.variants()[outs[-1].variant]
        vbytes = spmv_value_bytes(packed, shape) / max(packed.g.nnz, 1)
        smem_tbs = smem_model(st, packed, shape) / (k_ms * 1e-3) / 1e12
        prof = profiled_smem_pct(args.config) or {}
        smem = {"achieved_tbs": smem_tbs, "peak_tbs": smem_peak, "frac": smem_tbs / smem_peak,
                "model": f"corr_iters ({20 + vbytes:.1f} nnz + 40 d) + attempts 16 d bytes (engine.smem_model)",
                "value_bytes_per_nonzero": vbytes,
                "peak_source": f"128 B/clk/SM x {n_sm} SMs x {mhz} MHz (clock sampled under load)",
                "ncu_pipe_pct": prof.get("pct"), "ncu_source": prof.get("source"),
                "note": "the staged-operator SpMV streams an entry word, a gathered x and a dictionary value "
                        "(16 B; 8 B purely imaginary; none for the dominant value) per nonzero from shared memory; "
                        "ncu_pipe_pct is the measured l1tex shared-memory wavefront utilisation "
                        "of the committed capture (all shared-memory traffic, not the model's)"}

    # ---- end-to-end leg through the public API with host buffers ----------
    # every step: host problem -> HBM (qtm_problem_create), integrate the
    # shard, per-point sums + counters back to the host (and, for N>1, the
    # all-reduce in run_sharded), device buffers released
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if world > 1:
            run_sharded(packed, n_total, SEED, rank=rank, world_size=world, device=local,
                        on_failure="exclude", variant=args.variant)
        else:
            with DeviceProblem(packed, device=local, variant=args.variant) as dpe:
                o = dpe.run(SEED, 0, n_total, resident=True)
                if o.rc not in (0, -1, -4, -5, -6):
                    raise RuntimeError(o.error)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    e2e_value = (n_total - n_failed) / e2e_s
    n_out = packed.n_expect * packed.n_pts
    d2h = 8 * (2 * n_out + native.NSTATS + 2)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        sample = CPU_SAMPLE_PER_THREAD[args.config] * threads
        cval, _ = cpu_reference(packed, sample, 1, 0, threads)
        cpu = {"value": cval, "unit": "trajectories/s", "cores": threads, "kind": "port",
               "sample": f"{sample} trajectories of {args.config} (indices 0..{sample - 1}, "
                         f"Philox), oracle/mcwf_oracle.c, {threads} threads, one pass"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "trajectories/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64 (complex128)", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "config": args.config,
                       "trajectories": n_total, "trajectories_per_gpu": end - begin,
                       "seed": SEED, "stream": "philox", "rtol": packed.rtol,
                       "atol": packed.atol, "method": args.method,
                       "l2": "256 MiB buffer overwritten between timed steps",
                       "failed_trajectories": n_failed,
                       "failure_note": "reference-faithful OdeFailure(-5) step collapses, "
                                       "excluded from value and averages",
                       "kernel_variant": (native.variants()[outs[-1].variant]
                                          if outs[-1].variant >= 0 else "bdf_kernel"),
                       "grid_ctas": outs[-1].grid,
                       "history_rows": {"registers": layout["reg_rows"],
                                        "shared": layout["smem_rows"],
                                        "tmem": layout.get("tmem_rows", 0)},
                       "smem_per_cta": layout["smem_bytes"]},
            "e2e": {"value": e2e_value, "unit": "trajectories/s",
                    "h2d_bytes_per_step": int(packed.nbytes()), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": (profiled_traffic(args.config) or {}).get("bytes"),
                         "traffic_source": (profiled_traffic(args.config) or {}).get("source"),
                         "kernel": (("traj1_kernel (one thread per trajectory; state in registers)"
                                     if native.variant_small(outs[-1].variant)[0] else
                                     "traj_kernel (persistent; Nordsieck rows 2..7 + e buffers in "
                                     "TMEM, 2 CTAs/SM)" if layout.get("tmem_rows") else
                                     "traj_kernel (persistent; state in registers/smem)")
                                    if args.method == "adams" else
                                    "bdf_kernel (persistent; LU + Newton in smem/HBM workspace)"),
                         "peak_source": "measured DFMA throughput on this GPU "
                                        "(qtm_measure_fp64_peak, 2 flops/DFMA)",
                         "flops_per_launch": flops, "kernel_ms": k_ms,
                         "dmma_peak_tflops": dmma_peak,
                         "dmma_note": "measured FP64 tensor-core (mma.sync m8n8k4 DMMA) "
                                      "throughput: the ceiling of a dense H_eff path",
                         "build": ("fused multiply-add (QTM_FMAD=1, default)" if
                                   os.environ.get("QTM_LIB", "").find("parity") < 0 else
                                   "unfused parity build (QTM_FMAD=0)"),
                         "smem": smem,
                         "hbm_equiv_gbs": hbm_equiv,
                         "hbm_equiv_frac": hbm_equiv / hbm_peak if hbm_peak else None,
                         "hbm_peak_gbs": hbm_peak,
                         "hbm_equiv_note": "state-streaming model bytes (SURVEY §8d) / kernel "
                                           "time, against MEASURED_PEAKS.json hbm_gbs: the HBM "
                                           "bandwidth a design streaming the Nordsieck history "
                                           "would need to match this kernel; the kernel keeps "
                                           "state on chip, so the FP64 fraction is the bound"},
            "step_ms": [round(x, 3) for x in per_step],
            "work": {k: st[k] for k in ("attempts", "steps", "corr_iters", "jumps",
                                        "corr_fail", "err_reject", "overflow_attempts",
                                        "lu_factor")},
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
