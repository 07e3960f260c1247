"""Multi-GPU path logic on CPU: two gloo ranks run ``run_sharded`` with the
C oracle standing in for each rank's device run (the sharding rule, the
single all-reduce and the failure propagation are what is checked here; the
device engine itself is covered by the -m gpu tests)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _blocks(values, ok, block=256):
    """Stage 1 of the device's fixed-order reduction (ensemble_partial,
    qtm_capi.cu): per block of 256 trajectories, in trajectory order,
    skipping failed ones."""
    n = values.shape[0]
    nb = -(-n // block)
    bs = np.zeros((nb,) + values.shape[1:])
    bs2 = np.zeros((nb,) + values.shape[1:])
    for b in range(nb):
        s = np.zeros(values.shape[1:])
        s2 = np.zeros(values.shape[1:])
        for k in range(b * block, min(n, (b + 1) * block)):
            if ok[k]:
                s = s + values[k]
                s2 = s2 + values[k] * values[k]
        bs[b], bs2[b] = s, s2
    return bs, bs2


def _oracle_runner(packed, seed, begin, end, stream):
    from oracle import oracle
    from paper_1810_03047_b200.engine import RunOutput, combine_blocks
    r = oracle.run(packed, seed, begin, end, stream=stream, n_threads=2)
    ok = r["status"] == 0
    stats = np.zeros(16, np.int64)
    stats[:12] = r["stats"][ok].sum(axis=0)[:12]
    err = None
    if r["rc"]:
        err = dict(r["error"])
    bs, bs2 = _blocks(r["values"], ok)
    s, s2 = combine_blocks(bs, bs2)
    return RunOutput(s, s2, None, None, stats, None, None, None, None, err, r["rc"], 0.0, 0.0,
                     -1, 0, 0, end - begin, int((~ok).sum()), None, bs, bs2)


def _worker(rank, world, port, name, n, queue, max_steps, broken_rank=-1):
    import sys
    sys.path.insert(0, REPO)
    import dataclasses
    import torch.distributed as dist
    from paper_1810_03047_b200 import configs
    from paper_1810_03047_b200.engine import run_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = configs.build(name)
        if max_steps:
            p = dataclasses.replace(p, ode=dataclasses.replace(p.ode, max_steps=max_steps))
        runner = _oracle_runner if rank != broken_rank else _broken_runner
        res = run_sharded(p, n, 77, rank=rank, world_size=world, runner=runner)
        queue.put((rank, "ok", res.values, res.n_trajectories, res.stats, res.sumsq))
    except Exception as exc:  # noqa: BLE001
        queue.put((rank, "err", type(exc).__name__, str(exc), None, None))
    finally:
        dist.destroy_process_group()


def _broken_runner(packed, seed, begin, end, stream):
    raise RuntimeError("device setup failed on this rank")


def _spawn(name, n, world=2, max_steps=0, broken_rank=-1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n, q, max_steps, broken_rank))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda x: x[0])


def test_two_ranks_equal_single_process(oracle_lib):
    from paper_1810_03047_b200 import configs
    from paper_1810_03047_b200.packing import pack_problem
    out = _spawn("c2", 40)
    ref = oracle_lib.run(pack_problem(configs.build("c2")), 77, 0, 40)
    want = ref["values"].mean(axis=0)
    for rank, status, values, n, stats, _ in out:
        assert status == "ok", (status, values)
        assert n == 40
        np.testing.assert_allclose(values, want, rtol=0, atol=1e-13)
        assert stats["attempts"] == int(ref["stats"][:, 0].sum())


def test_failure_on_one_rank_raises_everywhere():
    # max_steps=1 makes every trajectory fail; the lowest failing index is
    # on rank 0, whose exception is the reference's OdeFailure text
    out = _spawn("c1", 8, max_steps=1)
    assert out[0][1] == "err" and out[0][2] == "OdeFailure"
    assert "ISTATE = -1" in out[0][3]
    assert out[1][1] == "err"


def test_sharded_sums_bitwise_invariant_to_rank_count():
    # block-aligned shards + one exact all-reduce of the block partials +
    # the device's block-order stage 2: 1, 2 and 3 ranks give identical bits
    # (600 trajectories = 3 blocks, the last one partial)
    outs = {w: _spawn("c1", 600, world=w) for w in (1, 2, 3)}
    for w in (2, 3):
        for rank in range(w):
            assert outs[w][rank][1] == "ok"
            np.testing.assert_array_equal(outs[w][rank][2], outs[1][0][2])
            np.testing.assert_array_equal(outs[w][rank][5], outs[1][0][5])


def test_setup_error_on_one_rank_does_not_hang():
    # rank 1 raises before integrating: it still joins the single collective,
    # so rank 0 learns of it and raises instead of waiting forever
    out = _spawn("c1", 300, broken_rank=1)
    assert out[1][1] == "err" and "device setup failed" in out[1][3]
    assert out[0][1] == "err" and "rank(s) [1]" in out[0][3]


def test_shard_ranges_are_block_aligned():
    from paper_1810_03047_b200.engine import shard_range
    for n, world in ((4096, 8), (100_000, 8), (500, 2), (600, 3), (10, 4), (257, 2)):
        ranges = [shard_range(n, world, r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        for (b0, e0), (b1, _) in zip(ranges, ranges[1:]):
            assert e0 == b1 and b1 % 256 in (0, n % 256) and b0 <= e0
    assert [shard_range(4096, 8, r) for r in range(8)] == [(512 * r, 512 * (r + 1)) for r in range(8)]


def test_bench_launcher_starts_ranks():
    """bench.py's own launcher (--gpus N outside torchrun) gives every rank
    the torchrun environment; 2 and 3 launched ranks reproduce the 1-rank
    sums bit for bit."""
    import json
    import subprocess
    import sys
    probe = os.path.join(REPO, "tests", "rank_probe.py")
    got = {}
    for n in (1, 2, 3):
        code = (f"import sys; sys.path.insert(0, {REPO!r}); import bench; "
                f"sys.exit(bench.launch_ranks([sys.executable, {probe!r}, '600'], {n}))")
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
        got[n] = json.loads(line)
        assert got[n]["world"] == n and got[n]["n"] == 600
    assert got[2]["sum"] == got[1]["sum"] == got[3]["sum"]
    assert got[2]["sumsq"] == got[1]["sumsq"] == got[3]["sumsq"]
