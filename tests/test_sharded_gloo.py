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


def _oracle_runner(packed, seed, begin, end, stream):
    from oracle import oracle
    from paper_1810_03047_b200.engine import RunOutput
    r = oracle.run(packed, seed, begin, end, stream=stream, n_threads=2)
    ok = r["status"] == 0
    vals = r["values"][ok]
    stats = np.zeros(16, np.int64)
    stats[:12] = r["stats"][ok].sum(axis=0)[:12]
    err = None
    if r["rc"]:
        err = dict(r["error"])
    return RunOutput(vals.sum(axis=0), (vals ** 2).sum(axis=0), None, None, stats, None, None,
                     None, None, err, r["rc"], 0.0, 0.0, -1, 0, 0, end - begin,
                     int((~ok).sum()))


def _worker(rank, world, port, name, n, queue, max_steps):
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
        res = run_sharded(p, n, 77, rank=rank, world_size=world, runner=_oracle_runner)
        queue.put((rank, "ok", res.values, res.n_trajectories, res.stats))
    except Exception as exc:  # noqa: BLE001
        queue.put((rank, "err", type(exc).__name__, str(exc), None))
    finally:
        dist.destroy_process_group()


def _spawn(name, n, world=2, max_steps=0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n, q, max_steps))
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
    for rank, status, values, n, stats in out:
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
