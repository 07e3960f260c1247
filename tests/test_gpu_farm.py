"""GPU worker and CLI on the device: the farm worker's
partial is the device ensemble over its global index range, checked
against the C oracle on the same streams; the CLI's inline and multi-GPU
modes write the reference's output format."""

import threading

import numpy as np
import pytest

from paper_1810_03047_b200 import cli, configs, farm
from paper_1810_03047_b200.packing import pack_problem

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method", ["adams", "bdf"])
def test_gpu_workers_match_oracle(method, oracle_lib):
    import dataclasses
    from paper_1810_03047_b200.problem import OdeConfig
    p = configs.build("c2", log_jumps=True)
    if method == "bdf":
        p = dataclasses.replace(p, ode=OdeConfig(method="bdf", rtol=p.ode.rtol, atol=p.ode.atol))
    pairs = [farm.QueueTransport.pair(timeout=300) for _ in range(2)]
    ths = [threading.Thread(target=farm.run_gpu_worker, args=(pairs[r][1], p, r))
           for r in range(2)]
    for t in ths:
        t.start()
    res = farm.run_master({r: pairs[r][0] for r in range(2)}, p, 65, 987654321)
    for t in ths:
        t.join(120)
    pk = pack_problem(p)
    parts = []
    for r, n in enumerate([33, 32]):
        b = farm.worker_stream_base(r)
        parts.append(oracle_lib.run(pk, 987654321, b, b + n, max_jumps=256))
    want = (33 * parts[0]["values"].mean(axis=0) + 32 * parts[1]["values"].mean(axis=0)) / 65
    assert res.n_trajectories == 65
    np.testing.assert_allclose(res.values, want, rtol=0, atol=1e-6)
    n_jumps = sum(int(q["jump_count"].sum()) for q in parts)
    assert len(res.jumps) == n_jumps


def test_cli_inline_and_two_device_split(tmp_path):
    out1, out2 = tmp_path / "a.csv", tmp_path / "b.csv"
    assert cli.main(["--problem", "photon", "--trajectories", "200", "--output", str(out1)]) == 0
    lines = out1.read_text().splitlines()
    assert lines[0] == "time,e0" and len(lines) == 1 + 201
    a = np.loadtxt(out1, delimiter=",", skiprows=1)
    # the K-device split integrates the same global trajectories; only the
    # order of the final summation differs
    import torch
    if torch.cuda.device_count() >= 2:
        assert cli.main(["--problem", "photon", "--trajectories", "200", "--gpus", "2",
                         "--output", str(out2)]) == 0
        b = np.loadtxt(out2, delimiter=",", skiprows=1)
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-14)
    assert a[0, 1] == 1.0  # <n> of |1> at t = 0


def test_cli_method_bdf(tmp_path, oracle_lib):
    out = tmp_path / "b.csv"
    assert cli.main(["--problem", "photon", "--trajectories", "64", "--method", "bdf",
                     "--output", str(out)]) == 0
    a = np.loadtxt(out, delimiter=",", skiprows=1)
    c = cli.parse_args(["--problem", "photon", "--method", "bdf"])
    ref = oracle_lib.run(pack_problem(cli.build_problem(c)), 987654321, 0, 64)
    np.testing.assert_allclose(a[:, 1], ref["values"].mean(axis=0)[0], rtol=0, atol=1e-6)


def test_cli_keep_trajectories(tmp_path):
    out = tmp_path / "u.csv"
    assert cli.main(["--problem", "unitary", "--trajectories", "4", "--steps", "20",
                     "--keep-trajectories", "--output", str(out)]) == 0
    mean = np.loadtxt(out, delimiter=",", skiprows=1)[:, 1]
    each = [np.loadtxt(f"{out}.trj{i}", delimiter=",", skiprows=1)[:, 1] for i in range(4)]
    np.testing.assert_allclose(np.mean(each, axis=0), mean, rtol=0, atol=1e-14)


def test_cli_numeric_failure_exit_code(capsys):
    rc = cli.main(["--problem", "jcm", "--steps", "1", "--t-to", "1e7", "--tol", "1e-8"])
    # no collapse channel ever restarts the segment, so a 1e7 horizon cannot
    # be reached: the run halts with the reference's OdeFailure (the oracle:
    # ISTATE -1, 50 000 steps exhausted near t = 823).  Which halt comes
    # first is itself ulp-sensitive in the reference algorithm (perturbing
    # its first step by a few ulp turns about half of these runs into a
    # step-size collapse, ISTATE -5 -- DESIGN.md), so only the mapping to
    # exit code 3 and the message are checked.
    assert rc == cli.EXIT_NUMERIC
    err = capsys.readouterr().err
    assert err.startswith("HALT: Error in ode solver, value ISTATE = ")
    assert "(inside trajectory)" in err
