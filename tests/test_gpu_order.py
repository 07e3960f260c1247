"""The processing order of a launch (longest expected trajectory first, by
the first jump threshold; qtm_capi.cu first_thresholds) changes when a
trajectory runs, never what it computes: per-trajectory series, jump logs,
counters and the ensemble sums are bitwise those of index order (QTM_ORDER=0)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(HERE, "tools", "lib_dump.py")

# more trajectories than resident CTAs, so the order is in effect
SPECS = ["c4:700:39", "c3:3000:12", "c2:4800:17", "c5:640:27", "c2+bdf:4000", "c4:600:39:lfsr113"]


@pytest.mark.gpu
def test_processing_order_does_not_change_results(tmp_path):
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"order{flag}.npz"
        env = dict(os.environ, QTM_ORDER=flag)
        r = subprocess.run([sys.executable, TOOL, "dump", str(out), *SPECS], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        outs.append(str(out))
    r = subprocess.run([sys.executable, TOOL, "cmp", *outs], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "RESULT: identical" in r.stdout
