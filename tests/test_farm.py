"""Farm protocol and CLI (host logic, no GPU): the GPU worker and master of
paper_1810_03047_b200/farm.py against the reference's own wire bytes and
digests (tests/golden/farm_wire.json, made by make_farm_golden.py), the
protocol end to end over in-process queues and TCP with the C oracle
standing in for the device run, and -- when /root/reference is present in
this container -- a REFERENCE master driving the GPU worker over TCP."""

import dataclasses
import json
import os
import sys
import threading
from types import SimpleNamespace

import numpy as np
import pytest

from paper_1810_03047_b200 import cli, configs, farm
from paper_1810_03047_b200.packing import pack_problem
from paper_1810_03047_b200.problem import TrajectoryResult
from paper_1810_03047_b200.problems import PROBLEM_BUILDERS

HERE = os.path.dirname(os.path.abspath(__file__))
WIRE = json.load(open(os.path.join(HERE, "golden", "farm_wire.json")))


# ---------------------------------------------------------------- digests
@pytest.mark.parametrize("name", sorted(PROBLEM_BUILDERS))
def test_cli_problem_digest_matches_reference(name):
    # equal digests <=> identical G, collapse/expect CSR arrays, psi0, grid
    # and ODE config (cluster.py:207-240), so these builders are bit-exact
    p = cli.build_problem(cli.RunConfig(problem=name, n_trajectories=1))
    assert farm.problem_digest(p) == int(WIRE["digests"][f"cli_{name}"])


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("log_jumps", [False, True])
def test_benchmark_config_digest_matches_reference(name, log_jumps):
    p = configs.build(name, log_jumps=log_jumps)
    assert farm.problem_digest(p) == int(WIRE["digests"][f"{name}_jumps{int(log_jumps)}"])


def test_digest_sees_every_field():
    p = configs.build("c1")
    d0 = farm.problem_digest(p)
    assert farm.problem_digest(dataclasses.replace(p, n_steps=p.n_steps + 1)) != d0
    assert farm.problem_digest(dataclasses.replace(
        p, ode=dataclasses.replace(p.ode, rtol=p.ode.rtol * 2))) != d0
    assert farm.problem_digest(dataclasses.replace(
        p, options=dataclasses.replace(p.options, log_jumps=True))) != d0


# ---------------------------------------------------------------- codec
def _golden_messages():
    times = np.linspace(0.0, 1.0, 3)
    vals = np.array([[0.25, -1.5, 3.0], [1e-300, np.pi, -0.0]])
    return {
        "hello": farm.Hello(3),
        "init": farm.Init(987654321, 0xFEDCBA9876543210, 17),
        "compute": farm.Compute(),
        "shutdown": farm.Shutdown(),
        "error": farm.Error(2, "numeric: trajectory 4 of rank 2: HALT é"),
        "result": farm.Result(TrajectoryResult(times, vals, 12, None)),
        "result_jumps": farm.Result(TrajectoryResult(times, vals, 5, [(0.125, 1), (0.5, 0)])),
    }


@pytest.mark.parametrize("key", ["hello", "init", "compute", "shutdown", "error", "result",
                                 "result_jumps"])
def test_encoding_is_byte_identical_to_reference(key):
    msg = _golden_messages()[key]
    raw = bytes.fromhex(WIRE["messages"][key])
    assert farm.encode_message(msg) == raw
    back = farm.decode_message(raw)
    assert type(back) is type(msg)
    if isinstance(msg, farm.Result):
        a, b = msg.partial, back.partial
        assert a.n_trajectories == b.n_trajectories and a.jumps == b.jumps
        assert np.array_equal(a.times, b.times)
        assert a.values.tobytes() == b.values.tobytes()  # -0.0 and 1e-300 survive
    else:
        assert back == msg


def test_decodes_a_reference_worker_partial():
    msg = farm.decode_message(bytes.fromhex(WIRE["messages"]["unitary_partial"]))
    r = msg.partial
    assert r.n_trajectories == 3 and r.values.shape == (1, 21)
    assert r.values[0, 0] == 1.0  # <sigma_z> of |0> at t = 0
    assert r.jumps is not None and all(k == 0 for _, k in r.jumps)
    assert farm.encode_message(msg).hex() == WIRE["messages"]["unitary_partial"]


def test_bad_frames_are_protocol_errors():
    with pytest.raises(farm.ClusterError, match="version"):
        farm.decode_message(b"\x02\x02")
    with pytest.raises(farm.ClusterError, match="tag"):
        farm.decode_message(b"\x01\x09")


# ---------------------------------------------------------------- protocol
def oracle_runner(problem, seed, begin, end, log_jumps):
    """The C oracle standing in for DeviceProblem.run (same global-index
    stream keying), returning the fields run_gpu_worker reads."""
    from oracle import oracle
    r = oracle.run(pack_problem(problem), seed, begin, end, n_threads=4, max_jumps=64)
    jumps = None
    if log_jumps and r["rc"] == 0:
        jumps = [(float(r["jump_t"][i, j]), int(r["jump_idx"][i, j]))
                 for i in range(end - begin) for j in range(int(r["jump_count"][i]))]
    return SimpleNamespace(rc=r["rc"], error=r["error"], sum=r["values"].sum(axis=0)), jumps


def _expected(problem, seed, counts):
    from oracle import oracle
    pk = pack_problem(problem)
    parts = []
    for rank, n in enumerate(counts):
        b = farm.worker_stream_base(rank)
        parts.append((n, oracle.run(pk, seed, b, b + n, n_threads=4)["values"].mean(axis=0)))
    total = sum(n for n, _ in parts)
    return sum(n * v for n, v in parts) / total


def _spawn_workers(problem, n, transports, runner=oracle_runner):
    ths = [threading.Thread(target=farm.run_gpu_worker, args=(transports[r], problem, r),
                            kwargs={"runner": runner}) for r in range(n)]
    for t in ths:
        t.start()
    return ths


def test_master_and_workers_over_queues(oracle_lib):
    p = configs.build("c1", log_jumps=True)
    pairs = [farm.QueueTransport.pair(timeout=120) for _ in range(3)]
    ths = _spawn_workers(p, 3, {r: pairs[r][1] for r in range(3)})
    res = farm.run_master({r: pairs[r][0] for r in range(3)}, p, 10, 77)
    for t in ths:
        t.join(60)
    assert res.n_trajectories == 10
    np.testing.assert_allclose(res.values, _expected(p, 77, [4, 3, 3]), rtol=0, atol=1e-13)
    assert res.jumps is not None and len(res.jumps) > 0


def test_master_and_workers_over_tcp(oracle_lib):
    p = PROBLEM_BUILDERS["photon"](n_steps=40)
    box = {}
    ready = threading.Event()

    def master():
        conns = farm.tcp_listen("127.0.0.1", 0, 2, timeout=60,
                                ready=lambda port: (box.__setitem__("port", port), ready.set()))
        try:
            box["res"] = farm.run_master(conns, p, 9, 5)
        finally:
            for c in conns.values():
                c.close()

    m = threading.Thread(target=master)
    m.start()
    assert ready.wait(30)
    ws = []
    for r in range(2):
        t = farm.tcp_connect("127.0.0.1", box["port"], r)
        th = threading.Thread(target=farm.run_gpu_worker, args=(t, p, r),
                              kwargs={"runner": oracle_runner})
        th.start()
        ws.append((t, th))
    m.join(120)
    for t, th in ws:
        th.join(60)
        t.close()
    np.testing.assert_allclose(box["res"].values, _expected(p, 5, [5, 4]), rtol=0, atol=1e-13)


def test_digest_mismatch_is_reported(oracle_lib):
    p = configs.build("c1")
    q = dataclasses.replace(p, n_steps=p.n_steps + 1)
    pairs = [farm.QueueTransport.pair(timeout=60) for _ in range(2)]
    ths = [threading.Thread(target=farm.run_gpu_worker, args=(pairs[r][1], q if r else p, r),
                            kwargs={"runner": oracle_runner}) for r in range(2)]
    for t in ths:
        t.start()
    with pytest.raises(farm.ClusterError) as ei:
        farm.run_master({r: pairs[r][0] for r in range(2)}, p, 4, 1)
    for t in ths:
        t.join(60)
    assert ei.value.kind == "digest" and "rank 1" in str(ei.value)


def test_numeric_failure_is_reported(oracle_lib):
    p = configs.build("c1")
    p = dataclasses.replace(p, ode=dataclasses.replace(p.ode, max_steps=1))
    a, b = farm.QueueTransport.pair(timeout=60)
    th = threading.Thread(target=farm.run_gpu_worker, args=(b, p, 0),
                          kwargs={"runner": oracle_runner})
    th.start()
    with pytest.raises(farm.ClusterError) as ei:
        farm.run_master({0: a}, p, 3, 1)
    th.join(60)
    assert ei.value.kind == "worker-numeric"
    assert "numeric: trajectory 0 of rank 0: HALT: Error in ode solver, value ISTATE = -1" \
        in str(ei.value)


def test_zero_assignment_returns_empty_partial():
    p = configs.build("c1")
    pairs = [farm.QueueTransport.pair(timeout=60) for _ in range(3)]
    ths = _spawn_workers(p, 3, {r: pairs[r][1] for r in range(3)},
                         runner=lambda *a: pytest.fail("no work expected"))
    # 0 trajectories cannot be requested from run_master; drive rank 2 by hand
    for r in range(3):
        pairs[r][0].send(farm.Init(1, farm.problem_digest(p), 0))
        pairs[r][0].send(farm.Compute())
    parts = [pairs[r][0].recv() for r in range(3)]
    for r in range(3):
        pairs[r][0].send(farm.Shutdown())
    for t in ths:
        t.join(60)
    assert all(isinstance(m, farm.Result) and m.partial.n_trajectories == 0 for m in parts)


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_reference_master_drives_gpu_worker(oracle_lib, tmp_path):
    """Interop: the reference's own TCP master (mcwf.cluster.run_master over
    tcp_listen) with one of its CPU workers and one GPU worker of this repo."""
    os.environ.setdefault("NUMBA_CACHE_DIR", str(tmp_path / "numba"))
    sys.path.insert(0, REF_SRC)
    try:
        from mcwf import cluster as rc
        from mcwf.problems import PROBLEM_BUILDERS as RB
    finally:
        sys.path.remove(REF_SRC)
    ref_p = RB["photon"](n_steps=20)
    ours = PROBLEM_BUILDERS["photon"](n_steps=20)
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    box = {}

    def master():
        conns = rc.tcp_listen("127.0.0.1", port, 2)
        try:
            box["res"] = rc.run_master(conns, ref_p, 6, 3)
        finally:
            for c in conns.values():
                c.close()

    m = threading.Thread(target=master)
    m.start()
    t0 = rc.tcp_connect("127.0.0.1", port, 0)          # reference CPU worker, rank 0
    w0 = threading.Thread(target=rc.run_worker, args=(t0, ref_p, 0))
    w0.start()
    t1 = farm.tcp_connect("127.0.0.1", port, 1)        # GPU worker (oracle stand-in), rank 1
    w1 = threading.Thread(target=farm.run_gpu_worker, args=(t1, ours, 1),
                          kwargs={"runner": oracle_runner})
    w1.start()
    m.join(300)
    for t, w in ((t0, w0), (t1, w1)):
        w.join(60)
        t.close()
    res = box["res"]
    assert res.n_trajectories == 6
    # rank 1's share (3 trajectories) is exactly what the GPU worker computed
    from oracle import oracle
    b = farm.worker_stream_base(1)
    mine = oracle.run(pack_problem(ours), 3, b, b + 3)["values"].mean(axis=0)
    # the reference master's average = (3 * rank0 + 3 * rank1) / 6
    rank0 = 2 * res.values - mine
    assert np.all(np.abs(rank0) <= 1.0 + 1e-12) and np.all(rank0 >= -1e-12)


# ---------------------------------------------------------------- CLI
def test_cli_usage_errors(capsys):
    assert cli.main(["--problem", "unitary", "--connect", "x:1"]) == cli.EXIT_USAGE
    assert cli.main(["--problem", "nope"]) == cli.EXIT_USAGE
    assert cli.main(["--problem", "unitary", "--listen", "127.0.0.1:1"]) == cli.EXIT_USAGE


def test_cli_method_bdf_builds_bdf_problems():
    for name in ("unitary", "c2"):
        c = cli.parse_args(["--problem", name, "--method", "bdf"])
        p = cli.build_problem(c)
        assert p.ode.method == "bdf" and p.ode.max_order == 6
        assert pack_problem(p).method == 1


def test_cli_defaults_follow_reference():
    c = cli.parse_args(["--problem", "jcm"])
    assert c.n_trajectories == 1 and c.tol == 1e-7 and c.seed == 987654321
    c = cli.parse_args(["--problem", "c4"])
    assert c.n_trajectories == 4096
    p = cli.build_problem(c)
    assert p.dim == 1024 and p.ode.rtol == 1e-8


def test_output_format(tmp_path):
    r = TrajectoryResult(np.array([0.0, 0.1]), np.array([[1.0, 1 / 3], [0.0, -2.5e-17]]), 2)
    f = tmp_path / "o.csv"
    cli.write_output(r, str(f), "csv")
    lines = f.read_text().splitlines()
    assert lines[0] == "time,e0,e1"
    assert lines[2] == "0.10000000000000001,0.33333333333333331,-2.4999999999999999e-17"
    assert float(lines[2].split(",")[1]) == 1 / 3  # 17 digits parse back exactly
    cli.write_output(r, str(f), "txt")
    assert f.read_text().splitlines()[0] == "0 1 0"
