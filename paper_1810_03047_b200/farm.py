"""GPU worker (and master) for the reference's trajectory farm protocol.

The reference distributes trajectories over a master and n workers that
talk through ordered point-to-point channels (``mcwf.cluster``,
/root/reference/pkg/src/mcwf/cluster.py).  A worker receives
Init(master_seed, problem digest, assigned count) and Compute, integrates
its assignment, and answers with ONE Result (its count-weighted partial
average) or ONE Error, then waits for Shutdown (cluster.py:395-427).  This
module speaks the same protocol with the same bytes on the wire (the TCP
frame format documented at cluster.py:13-26), so

  * ``run_gpu_worker`` can join a *reference* master (``mcwf --listen``)
    and integrate its share on a B200 instead of a CPU core, and
  * ``run_master`` (the same slot-table semantics as cluster.py:430-469)
    can drive reference CPU workers, GPU workers, or a mix.

Random streams.  A reference worker runs its assignment sequentially on
one stream derived from (master_seed, rank) (cluster.py:416-420), which no
parallel integrator can reproduce.  The GPU worker gives trajectory i of
rank r the per-trajectory stream of global index k = r * 2**32 + i (the
device's Philox or lfsr113 keying, csrc/qtm_rng.cuh), so its partial is a
deterministic function of (master_seed, rank, count) and statistically
equivalent to the reference's.

Everything on this path is host-side plumbing: the integration itself is
one ``DeviceProblem.run`` (the C ABI in include/qtm.h).
"""

from __future__ import annotations

import queue
import socket
import struct
import time
from dataclasses import dataclass
from hashlib import blake2b

import numpy as np

from .problem import ADAMS, TrajectoryResult, average_trajectories

__all__ = ["WIRE_VERSION", "Hello", "Init", "Compute", "Result", "Error", "Shutdown",
           "ClusterError", "TransportClosed", "encode_message", "decode_message",
           "problem_digest", "QueueTransport", "TcpTransport", "tcp_connect", "tcp_listen",
           "run_gpu_worker", "run_master", "worker_stream_base"]

WIRE_VERSION = 1
_RANK_STRIDE = 1 << 32  # global trajectory index = rank * 2**32 + i


# ------------------------------------------------------------------ messages
@dataclass(frozen=True)
class Hello:
    rank: int


@dataclass(frozen=True)
class Init:
    master_seed: int
    problem_digest: int
    assigned_count: int


@dataclass(frozen=True)
class Compute:
    pass


@dataclass(frozen=True)
class Result:
    partial: TrajectoryResult


@dataclass(frozen=True)
class Error:
    rank: int
    description: str


@dataclass(frozen=True)
class Shutdown:
    pass


class TransportClosed(Exception):
    """The peer went away (closed socket / queue, or a receive timeout)."""


class ClusterError(RuntimeError):
    """Farm failure; ``kind`` as in the reference: "worker-numeric",
    "digest", "transport" or "protocol"."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


# ------------------------------------------------------------------ codec
# payload := u8 version | u8 tag | body, little-endian (cluster.py:13-26)
_TAG_OF = {Hello: 0, Init: 1, Compute: 2, Result: 3, Error: 4, Shutdown: 5}
_RESULT_HEAD = struct.Struct("<IIQB")  # n_expect, n_points, n_trajectories, has_jumps
_JUMP = struct.Struct("<dI")           # (t*, channel)


def _result_body(r: TrajectoryResult) -> bytes:
    values = np.ascontiguousarray(r.values, dtype="<f8")
    n_expect, n_points = values.shape
    out = bytearray(_RESULT_HEAD.pack(n_expect, n_points, int(r.n_trajectories),
                                      int(r.jumps is not None)))
    out += np.ascontiguousarray(r.times, dtype="<f8").tobytes()
    out += values.tobytes()
    if r.jumps is not None:
        out += struct.pack("<I", len(r.jumps))
        for t, k in r.jumps:
            out += _JUMP.pack(float(t), int(k))
    return bytes(out)


def _parse_result(buf: bytes, pos: int) -> TrajectoryResult:
    n_expect, n_points, n_traj, has_jumps = _RESULT_HEAD.unpack_from(buf, pos)
    pos += _RESULT_HEAD.size
    times = np.frombuffer(buf, "<f8", n_points, pos).astype(np.float64)
    pos += 8 * n_points
    values = np.frombuffer(buf, "<f8", n_expect * n_points, pos).astype(np.float64)
    pos += 8 * n_expect * n_points
    jumps = None
    if has_jumps:
        (count,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        jumps = [(t, int(k)) for t, k in _JUMP.iter_unpack(buf[pos:pos + count * _JUMP.size])]
    return TrajectoryResult(times, values.reshape(n_expect, n_points), int(n_traj), jumps)


def encode_message(msg) -> bytes:
    """Payload bytes of one message (cluster.py:152-168 layout)."""
    try:
        tag = _TAG_OF[type(msg)]
    except KeyError:
        raise TypeError(f"not a farm message: {msg!r}") from None
    head = bytes((WIRE_VERSION, tag))
    if tag == 0:
        return head + struct.pack("<I", msg.rank)
    if tag == 1:
        return head + struct.pack("<QQI", msg.master_seed, msg.problem_digest,
                                  msg.assigned_count)
    if tag == 3:
        return head + _result_body(msg.partial)
    if tag == 4:
        text = msg.description.encode("utf-8")
        return head + struct.pack("<II", msg.rank, len(text)) + text
    return head  # Compute, Shutdown: empty body


def decode_message(payload: bytes):
    if len(payload) < 2:
        raise ClusterError("protocol", "truncated message")
    version, tag = payload[0], payload[1]
    if version != WIRE_VERSION:
        raise ClusterError("protocol", f"unsupported wire version {version}")
    if tag == 0:
        return Hello(struct.unpack_from("<I", payload, 2)[0])
    if tag == 1:
        seed, digest, count = struct.unpack_from("<QQI", payload, 2)
        return Init(seed, digest, count)
    if tag == 2:
        return Compute()
    if tag == 3:
        return Result(_parse_result(payload, 2))
    if tag == 4:
        rank, n = struct.unpack_from("<II", payload, 2)
        return Error(rank, payload[10:10 + n].decode("utf-8"))
    if tag == 5:
        return Shutdown()
    raise ClusterError("protocol", f"unknown message tag {tag}")


# ------------------------------------------------------------------ digest
def _csr_bytes(m) -> list[bytes]:
    return [struct.pack("<I", m.n),
            np.ascontiguousarray(m.row_ptr, dtype="<i8").tobytes(),
            np.ascontiguousarray(m.col_ind, dtype="<i8").tobytes(),
            np.ascontiguousarray(m.values, dtype="<c16").tobytes()]


def problem_digest(problem) -> int:
    """64-bit BLAKE2b digest of the problem definition, byte-compatible
    with the reference's (cluster.py:207-240): magic, grid, ODE config,
    jump-log flag, G (or a callback marker), collapse and expectation
    operators, psi0."""
    ode = problem.ode
    init = np.nan if ode.initial_step is None else float(ode.initial_step)
    chunks = [b"MCWFPROB1",
              struct.pack("<IddI", problem.dim, problem.t_from, problem.t_to, problem.n_steps),
              struct.pack("<BddIQd", 0 if ode.method == ADAMS else 1, ode.rtol, ode.atol,
                          ode.max_order, ode.max_steps, init),
              struct.pack("<B", 1 if problem.options.log_jumps else 0)]
    if problem.generator is None:
        chunks.append(b"\x01")
    else:
        chunks.append(b"\x00")
        chunks += _csr_bytes(problem.generator.g)
    for ops in (problem.collapse_csr, problem.expect_csr):
        chunks.append(struct.pack("<I", len(ops)))
        for m in ops:
            chunks += _csr_bytes(m)
    chunks.append(np.ascontiguousarray(problem.psi0, dtype="<c16").tobytes())
    h = blake2b(digest_size=8)
    for c in chunks:
        h.update(c)
    return int.from_bytes(h.digest(), "little")


# ------------------------------------------------------------------ transports
class QueueTransport:
    """In-process channel (message objects through a pair of queues)."""

    _EOF = object()

    def __init__(self, inbox, outbox, timeout: float | None = None):
        self._in, self._out, self._timeout = inbox, outbox, timeout

    @classmethod
    def pair(cls, timeout: float | None = None):
        a, b = queue.Queue(), queue.Queue()
        return cls(a, b, timeout), cls(b, a, timeout)

    def send(self, msg):
        self._out.put(msg)

    def recv(self):
        try:
            item = self._in.get(timeout=self._timeout)
        except queue.Empty:
            raise TransportClosed from None
        if item is self._EOF:
            raise TransportClosed
        return item

    def close(self):
        self._out.put(self._EOF)


class TcpTransport:
    """Length-prefixed frames (u32 length | payload) over a stream socket."""

    def __init__(self, sock: socket.socket, timeout: float = 600.0):
        self._sock = sock
        sock.settimeout(timeout)

    def send(self, msg):
        data = encode_message(msg)
        self._sock.sendall(struct.pack("<I", len(data)) + data)

    def _read(self, n: int) -> bytes:
        buf = bytearray()
        while len(buf) < n:
            try:
                part = self._sock.recv(n - len(buf))
            except OSError as exc:  # includes socket.timeout
                raise TransportClosed from exc
            if not part:
                raise TransportClosed
            buf += part
        return bytes(buf)

    def recv(self):
        (n,) = struct.unpack("<I", self._read(4))
        return decode_message(self._read(n))

    def close(self):
        try:
            self._sock.shutdown(socket.SHUT_RDWR)
        except OSError:
            pass
        self._sock.close()


def tcp_connect(host: str, port: int, rank: int, retry_for: float = 60.0) -> TcpTransport:
    """Worker side: connect (retrying while the master starts) and announce
    the rank with Hello."""
    deadline = time.monotonic() + retry_for
    while True:
        try:
            sock = socket.create_connection((host, port), timeout=10.0)
            break
        except OSError as exc:
            if time.monotonic() > deadline:
                raise ClusterError("transport",
                                   f"cannot reach master at {host}:{port}: {exc}") from exc
            time.sleep(0.05)
    t = TcpTransport(sock)
    t.send(Hello(rank))
    return t


def tcp_listen(host: str, port: int, n_workers: int, timeout: float = 600.0,
               ready=None) -> dict:
    """Master side: accept n_workers connections keyed by their Hello rank.
    ``ready(port)`` (optional) is called once the socket listens (port 0
    binds an ephemeral port)."""
    srv = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
    srv.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
    srv.bind((host, port))
    srv.listen(n_workers)
    srv.settimeout(timeout)
    if ready is not None:
        ready(srv.getsockname()[1])
    conns: dict = {}
    try:
        while len(conns) < n_workers:
            try:
                sock, _ = srv.accept()
            except socket.timeout as exc:
                raise ClusterError("transport", "timed out waiting for workers") from exc
            t = TcpTransport(sock)
            hello = t.recv()
            if not isinstance(hello, Hello):
                raise ClusterError("protocol", f"expected Hello, got {hello!r}")
            if not 0 <= hello.rank < n_workers or hello.rank in conns:
                raise ClusterError("protocol", f"bad worker rank {hello.rank}")
            conns[hello.rank] = t
    finally:
        srv.close()
    return conns


# ------------------------------------------------------------------ worker
def worker_stream_base(rank: int) -> int:
    """Global trajectory index of a GPU worker's first trajectory."""
    return rank * _RANK_STRIDE


def _zero_partial(problem) -> TrajectoryResult:
    times = problem.time_grid()
    return TrajectoryResult(times, np.zeros((len(problem.expect_csr), times.shape[0])), 0,
                            [] if problem.options.log_jumps else None)


def _drain_until_shutdown(transport) -> None:
    try:
        while not isinstance(transport.recv(), Shutdown):
            pass
    except TransportClosed:
        pass


def _device_runner(device: int, stream: str, max_jumps: int):
    def run(problem, seed, begin, end, log_jumps):
        from .engine import DeviceProblem, _jump_list, run_logged
        with DeviceProblem(problem, device=device) as dp:
            if log_jumps:
                out = run_logged(dp, seed, begin, end, stream=stream, max_jumps=max_jumps)
            else:
                out = dp.run(seed, begin, end, stream=stream, per_trajectory=False)
        return out, (_jump_list(out) if log_jumps and out.rc == 0 else None)
    return run


def run_gpu_worker(transport, problem, rank: int, *, device: int = 0, stream: str = "philox",
                   max_jumps: int = 1024, runner=None) -> None:
    """One farm worker on one GPU, protocol-compatible with the reference
    worker loop (cluster.py:395-427): Init (digest check), Compute, one
    Result or Error, then wait for Shutdown.

    ``runner(problem, seed, begin, end, log_jumps) -> (RunOutput, jumps)``
    defaults to the device engine; the CPU tests inject the oracle."""
    try:
        init = transport.recv()
    except TransportClosed:
        return
    if not isinstance(init, Init):
        transport.send(Error(rank, f"protocol: expected Init, got {type(init).__name__}"))
        return _drain_until_shutdown(transport)
    if init.problem_digest != problem_digest(problem):
        transport.send(Error(rank, "digest: problem definition mismatch with master"))
        return _drain_until_shutdown(transport)
    try:
        msg = transport.recv()
    except TransportClosed:
        return
    if not isinstance(msg, Compute):
        transport.send(Error(rank, f"protocol: expected Compute, got {type(msg).__name__}"))
        return _drain_until_shutdown(transport)

    count = init.assigned_count
    if count == 0:
        transport.send(Result(_zero_partial(problem)))
        return _drain_until_shutdown(transport)
    from .engine import raise_for_status
    run = runner or _device_runner(device, stream, max_jumps)
    base = worker_stream_base(rank)
    log_jumps = bool(problem.options.log_jumps)
    out, jumps = run(problem, init.master_seed, base, base + count, log_jumps)
    if out.rc != 0:
        # the lowest failing trajectory, with the reference's message text
        local = int(out.error["traj"]) - base
        try:
            raise_for_status(out.rc, out.error, problem)
            text = f"trajectory failed with status {out.rc}"
        except (RuntimeError, ValueError) as exc:
            text = str(exc)
        transport.send(Error(rank, f"numeric: trajectory {local} of rank {rank}: {text}"))
        return _drain_until_shutdown(transport)
    times = problem.time_grid()
    transport.send(Result(TrajectoryResult(times, out.sum / count, count, jumps)))
    return _drain_until_shutdown(transport)


# ------------------------------------------------------------------ master
def run_master(transports: dict, problem, n_total: int, master_seed: int) -> TrajectoryResult:
    """Coordinate one farm run (cluster.py:430-469 semantics): Init and
    Compute to every rank, exactly one reply per rank read in rank order,
    Shutdown to all, partials averaged in rank order (so the result does
    not depend on arrival order)."""
    from .engine import partition_trajectories
    ranks = sorted(transports)
    counts = partition_trajectories(n_total, len(ranks))
    digest = problem_digest(problem)
    partials: dict = {}
    errors: list = []
    try:
        for r in ranks:
            transports[r].send(Init(master_seed, digest, counts[r]))
        for r in ranks:
            transports[r].send(Compute())
        for r in ranks:
            msg = transports[r].recv()
            if isinstance(msg, Result):
                if msg.partial.n_trajectories != counts[r]:
                    raise ClusterError("protocol",
                                       f"rank {r} returned {msg.partial.n_trajectories} "
                                       f"trajectories, assigned {counts[r]}")
                partials[r] = msg.partial
            elif isinstance(msg, Error):
                errors.append(msg)
            else:
                raise ClusterError("protocol", f"unexpected message from rank {r}: {msg!r}")
    except TransportClosed as exc:
        raise ClusterError("transport", "worker channel closed before its result arrived") \
            from exc
    finally:
        for r in ranks:
            try:
                transports[r].send(Shutdown())
            except (TransportClosed, OSError):
                pass
    if errors:
        detail = "; ".join(f"rank {e.rank}: {e.description}" for e in errors)
        if all(e.description.startswith("numeric:") for e in errors):
            kind = "worker-numeric"
        elif any("digest:" in e.description for e in errors):
            kind = "digest"
        else:
            kind = "protocol"
        raise ClusterError(kind, f"{len(errors)} worker(s) failed: {detail}")
    return average_trajectories([partials[r] for r in ranks])
