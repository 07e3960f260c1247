"""Command line: the reference CLI's run modes on B200s.

Mirrors ``mcwf`` (/root/reference/pkg/src/mcwf/cli.py): the same problem
names, options, CSV/text output (17 significant digits, header
``time,e0,e1,...``) and exit codes (0 ok, 2 usage, 3 numeric failure,
4 transport failure), with the CPU trajectory loop replaced by the device
engine:

    python -m paper_1810_03047_b200.cli --problem unitary --trajectories 1000
    python -m paper_1810_03047_b200.cli --problem c4 --gpus 8
    # GPU worker for a reference master started with
    #   mcwf --problem unitary --listen 0.0.0.0:7000 --expect-workers 2
    python -m paper_1810_03047_b200.cli --problem unitary --connect host:7000 --rank 1
    # master for any mix of reference CPU workers and GPU workers
    python -m paper_1810_03047_b200.cli --problem unitary --listen 0.0.0.0:7000 \\
        --expect-workers 2

Inline and ``--gpus K`` runs integrate global trajectories 0..N-1 with the
per-trajectory streams of the device (``--stream philox|lfsr113``); K GPUs
take contiguous index ranges (one host thread per device; the C ABI runs
without the GIL) and their sums are combined in device order.
``--method bdf`` runs the BDF kernel (modified Newton with a per-trajectory
LU, csrc/qtm_bdf.cuh).  ``--local-workers`` (the reference's CPU process
farm) is not offered: there is no CPU path here.
"""

from __future__ import annotations

import argparse
import os
import sys
import threading
from dataclasses import dataclass

import numpy as np

from . import configs, farm
from .problem import ADAMS, BDF, OdeConfig, OdeFailure, RunOptions, TrajectoryResult
from .problems import PROBLEM_BUILDERS, PROBLEM_DEFAULTS

__all__ = ["RunConfig", "build_problem", "run", "run_local_gpus", "write_output", "main",
           "parse_args"]

EXIT_OK, EXIT_USAGE, EXIT_NUMERIC, EXIT_TRANSPORT = 0, 2, 3, 4
DEFAULT_SEED = 987654321
_BENCH = {name: (None, None, configs.N_TRAJECTORIES[name]) for name in configs.CONFIGS}


@dataclass
class RunConfig:
    problem: str
    n_trajectories: int
    t_from: float = 0.0
    t_to: float | None = None
    n_steps: int | None = None
    method: str = ADAMS
    tol: float = 1e-7
    seed: int = DEFAULT_SEED
    output: str = "-"
    fmt: str = "csv"
    gpus: int = 1
    device: int = 0
    stream: str = "philox"
    listen: str | None = None
    expect_workers: int | None = None
    connect: str | None = None
    rank: int | None = None
    only_final_trj: bool = True
    verbose: bool = False


def build_problem(config: RunConfig):
    """The named problem with the CLI's grid and tolerance overrides (same
    construction as the reference CLI, cli.py:52-63); c1..c5 are the
    benchmark configs, whose own grids and tolerances apply unless
    overridden."""
    if config.method not in (ADAMS, BDF):
        raise ValueError(f"unknown method {config.method!r}")
    options = RunOptions(only_final_trj=config.only_final_trj, output_target=config.output,
                         verbose=config.verbose)
    if config.problem in PROBLEM_BUILDERS:
        n_steps, t_to, _ = PROBLEM_DEFAULTS[config.problem]
        return PROBLEM_BUILDERS[config.problem](
            n_steps=config.n_steps if config.n_steps is not None else n_steps,
            t_from=config.t_from, t_to=config.t_to if config.t_to is not None else t_to,
            ode=OdeConfig(method=config.method, rtol=config.tol), options=options)
    if config.problem in configs.CONFIGS:
        import dataclasses
        p = configs.build(config.problem)
        if config.method != ADAMS:
            p = dataclasses.replace(p, ode=OdeConfig(method=config.method, rtol=p.ode.rtol,
                                                     atol=p.ode.atol))
        return dataclasses.replace(
            p, options=options, t_from=config.t_from,
            t_to=config.t_to if config.t_to is not None else p.t_to,
            n_steps=config.n_steps if config.n_steps is not None else p.n_steps)
    raise ValueError(f"unknown problem {config.problem!r}")


def _rows(result: TrajectoryResult, fmt: str) -> str:
    if fmt not in ("csv", "txt"):
        raise ValueError(f"unknown output format {fmt!r}")
    sep = "," if fmt == "csv" else " "
    n_e = result.values.shape[0]
    lines = ["time," + ",".join(f"e{k}" for k in range(n_e))] if fmt == "csv" else []
    for j, t in enumerate(result.times):
        lines.append(sep.join([f"{t:.17g}"] + [f"{result.values[k, j]:.17g}"
                                               for k in range(n_e)]))
    return "\n".join(lines) + "\n"


def write_output(result: TrajectoryResult, target: str, fmt: str = "csv") -> None:
    text = _rows(result, fmt)
    if target == "-":
        sys.stdout.write(text)
        return
    try:
        with open(target, "w", newline="") as fh:
            fh.write(text)
    except OSError as exc:
        raise OSError(f"cannot write output file {target!r}: {exc}") from exc


def _resolve_output(path: str) -> str:
    base = os.environ.get("MCWF_OUTPUT_DIR")
    if path != "-" and base and not os.path.isabs(path):
        return os.path.join(base, path)
    return path


def _hostport(spec: str) -> tuple[str, int]:
    host, sep, port = spec.rpartition(":")
    if not sep or not host:
        raise ValueError(f"expected HOST:PORT, got {spec!r}")
    return host, int(port)


def _say(config: RunConfig, msg: str) -> None:
    if config.verbose:
        print(msg, file=sys.stderr)


def run_local_gpus(problem, n_total: int, seed: int, n_gpus: int, *, first_device: int = 0,
                   stream: str = "philox", keep: bool = False):
    """Trajectories 0..n_total-1 over n_gpus devices (contiguous ranges, one
    host thread per device).  Returns (TrajectoryResult, per-trajectory
    series or None).  Raises the reference exception of the lowest failing
    trajectory."""
    from .engine import DeviceProblem, partition_trajectories, raise_for_status
    from .packing import pack_problem
    packed = pack_problem(problem)
    counts = partition_trajectories(n_total, n_gpus)
    starts = np.concatenate([[0], np.cumsum(counts)]).astype(int)
    outs: list = [None] * n_gpus
    errs: list = [None] * n_gpus

    def work(g):
        try:
            with DeviceProblem(packed, device=first_device + g) as dp:
                outs[g] = dp.run(seed, int(starts[g]), int(starts[g + 1]), stream=stream,
                                 per_trajectory=keep, resident=not keep)
        except Exception as exc:  # noqa: BLE001 - re-raised on the caller's thread
            errs[g] = exc

    threads = [threading.Thread(target=work, args=(g,)) for g in range(n_gpus) if counts[g]]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    done = [o for o in outs if o is not None]
    for o in done:  # lowest global index first: devices are in index order
        if o.rc != 0:
            raise_for_status(o.rc, o.error)
    total = sum(o.sum for o in done)
    result = TrajectoryResult(packed.times, total / n_total, n_total, None)
    series = np.concatenate([o.values for o in done]) if keep else None
    return result, series


def _run_worker(config: RunConfig) -> int:
    host, port = _hostport(config.connect)
    problem = build_problem(config)
    _say(config, f"GPU worker rank {config.rank} (device {config.device}) -> {host}:{port}")
    t = farm.tcp_connect(host, port, config.rank)
    try:
        farm.run_gpu_worker(t, problem, config.rank, device=config.device, stream=config.stream)
    finally:
        t.close()
    return EXIT_OK


def run(config: RunConfig) -> int:
    """Execute one CLI run; returns the process exit code."""
    try:
        if config.connect is not None:
            return _run_worker(config)
        problem = build_problem(config)
        target = _resolve_output(config.output)
        if config.listen is not None:
            if not config.expect_workers:
                raise ValueError("--listen requires --expect-workers")
            host, port = _hostport(config.listen)
            _say(config, f"master on {host}:{port}, waiting for {config.expect_workers} workers")
            conns = farm.tcp_listen(host, port, config.expect_workers)
            try:
                result = farm.run_master(conns, problem, config.n_trajectories, config.seed)
            finally:
                for c in conns.values():
                    c.close()
        else:
            keep = not config.only_final_trj
            if keep and target == "-":
                raise ValueError("--keep-trajectories needs a file output target")
            _say(config, f"{config.n_trajectories} trajectories on {config.gpus} GPU(s), "
                         f"seed {config.seed}")
            result, series = run_local_gpus(problem, config.n_trajectories, config.seed,
                                            config.gpus, first_device=config.device,
                                            stream=config.stream, keep=keep)
            if keep:
                for i, v in enumerate(series):
                    write_output(TrajectoryResult(result.times, v, 1, None),
                                 f"{target}.trj{i}", config.fmt)
        write_output(result, target, config.fmt)
        return EXIT_OK
    except OdeFailure as exc:
        print(str(exc), file=sys.stderr)
        return EXIT_NUMERIC
    except farm.ClusterError as exc:
        print(f"HALT: cluster failure ({exc.kind}): {exc}", file=sys.stderr)
        return EXIT_NUMERIC if exc.kind == "worker-numeric" else EXIT_TRANSPORT
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_TRANSPORT


def _positive(text: str) -> int:
    v = int(text)
    if v < 1:
        raise argparse.ArgumentTypeError(f"expected a positive integer, got {v}")
    return v


def _parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(
        prog="qtm-b200", description="Quantum-trajectory (MCWF) ensembles on B200 GPUs; "
                                     "command line of the reference mcwf.")
    names = sorted(PROBLEM_BUILDERS) + sorted(configs.CONFIGS)
    p.add_argument("--problem", required=True, choices=names)
    p.add_argument("--trajectories", type=_positive, default=None)
    p.add_argument("--t-from", type=float, default=0.0)
    p.add_argument("--t-to", type=float, default=None)
    p.add_argument("--steps", type=_positive, default=None)
    p.add_argument("--method", choices=[ADAMS, BDF], default=ADAMS)
    p.add_argument("--tol", type=float, default=1e-7)
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--output", default="-", metavar="PATH")
    p.add_argument("--format", choices=["csv", "txt"], default="csv", dest="fmt")
    p.add_argument("--gpus", type=_positive, default=1, metavar="K",
                   help="integrate on K local GPUs (default 1)")
    p.add_argument("--device", type=int, default=None,
                   help="first CUDA device (default $LOCAL_RANK or 0)")
    p.add_argument("--stream", choices=["philox", "lfsr113"], default="philox")
    p.add_argument("--listen", metavar="HOST:PORT")
    p.add_argument("--expect-workers", type=_positive, default=None)
    p.add_argument("--connect", metavar="HOST:PORT")
    p.add_argument("--rank", type=int, default=None)
    p.add_argument("--keep-trajectories", action="store_true")
    p.add_argument("--verbose", action="store_true")
    return p


def parse_args(argv=None) -> RunConfig:
    ns = _parser().parse_args(argv)
    if ns.connect is not None and ns.rank is None:
        _parser().error("--connect requires --rank")
    seed = ns.seed if ns.seed is not None else int(os.environ.get("MCWF_SEED", DEFAULT_SEED))
    defaults = PROBLEM_DEFAULTS.get(ns.problem) or _BENCH[ns.problem]
    tol = ns.tol
    device = ns.device if ns.device is not None else int(os.environ.get("LOCAL_RANK", 0))
    return RunConfig(problem=ns.problem,
                     n_trajectories=ns.trajectories or defaults[2],
                     t_from=ns.t_from, t_to=ns.t_to, n_steps=ns.steps, method=ns.method,
                     tol=tol, seed=seed, output=ns.output, fmt=ns.fmt, gpus=ns.gpus,
                     device=device, stream=ns.stream, listen=ns.listen,
                     expect_workers=ns.expect_workers, connect=ns.connect, rank=ns.rank,
                     only_final_trj=not ns.keep_trajectories, verbose=ns.verbose)


def main(argv=None) -> int:
    try:
        config = parse_args(argv)
    except SystemExit as exc:
        return int(exc.code) if exc.code is not None else EXIT_USAGE
    return run(config)


if __name__ == "__main__":
    sys.exit(main())
