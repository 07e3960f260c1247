"""The value encodings of the staged sliced-ELL copy of G on the wide kernel
variants (csrc/qtm_capi.cu build_sell, csrc/qtm_traj.cuh sell_val_flag): the
dominant purely imaginary value served from the kernel parameters (c4: every
off-diagonal of the Ising chain), the other purely imaginary values as 8-byte
loads with the diagonal aligned per warp by inserted exact zeros (c5).  They
change how a value reaches the multiply, never the bits multiplied or the
order of a row's sum (reference _kernels.py:150-154): per-trajectory series,
jump logs, counters and ensemble sums are bitwise those of the plain encoding
(QTM_DOM=0), variant by variant."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(HERE, "tools", "lib_dump.py")

# c4 on the TMEM and register variants (dominant value), c5 on both of its
# shapes (8-byte values, aligned diagonal), c2 / c3 forced onto wide variants
# (ragged rows: padding and inserted zeros in play), LFSR113 streams once
SPECS = ["c4:300:39", "c4:150:22", "c5:96:39", "c5:96:27", "c5:64:26", "c3:128:6", "c2:128:6",
         "c4:160:39:lfsr113"]


@pytest.mark.gpu
def test_value_encodings_do_not_change_results(tmp_path):
    outs = {}
    for flag in ("0", "1", "2", "3"):
        out = tmp_path / f"dom{flag}.npz"
        env = dict(os.environ, QTM_DOM=flag)
        r = subprocess.run([sys.executable, TOOL, "dump", str(out), *SPECS], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        outs[flag] = str(out)
    for flag in ("1", "2", "3"):
        r = subprocess.run([sys.executable, TOOL, "cmp", outs["0"], outs[flag]],
                           capture_output=True, text=True, timeout=300)
        print(f"QTM_DOM={flag}:", r.stdout.strip().splitlines()[-1])
        assert r.returncode == 0, r.stdout + r.stderr
        assert "RESULT: identical" in r.stdout
