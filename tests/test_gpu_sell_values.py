"""The value encodings of the staged sliced-ELL copy of G on the wide kernel
variants (csrc/qtm_capi.cu build_sell, csrc/qtm_traj.cuh sell_val_flag): the
dominant purely imaginary value served from the kernel parameters (c4: every
off-diagonal of the Ising chain), the other purely imaginary values as 8-byte
loads with the diagonal aligned per warp by inserted exact zeros (c5).  They
change how a value reaches the multiply, never the bits multiplied or the
order of a row's sum (reference _kernels.py:150-154): per-trajectory series,
jump logs, counters and ensemble sums are bitwise those of the plain encoding
(QTM_DOM=0), variant by variant.  The same holds for the table-free form of a
time-dependent term whose entries all hold one value (c4td, QTM_DOM bit 2)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(HERE, "tools", "lib_dump.py")

# c4 on the TMEM and register variants (dominant value), c5 on both of its
# shapes (8-byte values, aligned diagonal), c2 / c3 forced onto wide variants
# (ragged rows: padding and inserted zeros in play), LFSR113 streams once
# c4td on two time-dependent variants (the single-valued term without tables)
SPECS = ["c4:300:39", "c4:150:22", "c5:96:39", "c5:96:27", "c5:64:26", "c3:128:6", "c2:128:6",
         "c4:160:39:lfsr113", "c4td:150:36", "c4td:100:34"]


@pytest.mark.gpu
def test_value_encodings_do_not_change_results(tmp_path):
    outs = {}
    for flag in ("0", "1", "2", "3", "7"):
        out = tmp_path / f"dom{flag}.npz"
        env = dict(os.environ, QTM_DOM=flag)
        r = subprocess.run([sys.executable, TOOL, "dump", str(out), *SPECS], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        outs[flag] = str(out)
    for flag in ("1", "2", "3", "7"):
        r = subprocess.run([sys.executable, TOOL, "cmp", outs["0"], outs[flag]],
                           capture_output=True, text=True, timeout=300)
        print(f"QTM_DOM={flag}:", r.stdout.strip().splitlines()[-1])
        assert r.returncode == 0, r.stdout + r.stderr
        assert "RESULT: identical" in r.stdout


def _random_problem(kind, d=300, seed=5):
    """Sparse random operators whose G exercises the staging rules: `real` --
    real H off-diagonals with many distinct values (purely imaginary G entries,
    8-byte values, ragged rows, some rows without a stored diagonal); `dominant`
    -- one value on most off-diagonals plus a few others; `complex` -- complex
    H off-diagonals (nothing to encode: the plain loop)."""
    import numpy as np

    from paper_1810_03047_b200.problem import OdeConfig, QuantumProblem, RunOptions
    from paper_1810_03047_b200.qops import OperatorSet

    rng = np.random.default_rng(seed)
    h = np.zeros((d, d), dtype=np.complex128)
    for i in range(d):
        for off in (1, 7, 31):
            j = i + off
            if j >= d or rng.random() < 0.25:
                continue
            if kind == "real":
                v = rng.uniform(0.1, 0.6)
            elif kind == "dominant":
                v = 0.35 if rng.random() < 0.8 else rng.uniform(0.1, 0.6)
            else:
                v = rng.uniform(0.1, 0.6) + 1j * rng.uniform(-0.3, 0.3)
            h[i, j] = v
            h[j, i] = np.conj(v)
    diag = rng.uniform(-1.0, 1.0, d)
    diag[rng.random(d) < 0.1] = 0.0  # rows of G without a stored diagonal (where the decay is 0 too)
    h += np.diag(diag)
    c = np.zeros((d, d), dtype=np.complex128)
    for i in range(1, d, 2):  # every other level decays: the others have no -C^+C/2 on the diagonal
        c[i - 1, i] = np.sqrt(1.5)
    obs = np.diag(np.arange(d, dtype=np.float64)).astype(np.complex128)
    psi0 = rng.normal(size=d) + 1j * rng.normal(size=d)
    psi0 /= np.linalg.norm(psi0)
    return QuantumProblem.from_operators(OperatorSet(h, (c,), (obs,)), psi0, 0.0, 2.0, 20,
                                         ode=OdeConfig(rtol=1e-8, atol=1e-10),
                                         options=RunOptions(log_jumps=True))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["real", "dominant", "complex"])
@pytest.mark.parametrize("variant", [39, 27])
def test_value_encodings_on_random_operators(kind, variant, oracle_lib, monkeypatch):
    """Random sparse operators on the wide variants: every encoding gives the
    bits of the plain one, and the plain one matches the C oracle."""
    import numpy as np

    from paper_1810_03047_b200.engine import DeviceProblem
    from paper_1810_03047_b200.packing import pack_problem

    pk = pack_problem(_random_problem(kind))
    n, seed = 24, 987654321
    outs = {}
    for flag in ("0", "1", "2", "3"):
        monkeypatch.setenv("QTM_DOM", flag)
        with DeviceProblem(pk, variant=variant) as dp:
            outs[flag] = dp.run(seed, 0, n, max_jumps=64)
        assert outs[flag].rc == 0, outs[flag].error
    base = outs["0"]
    for flag in ("1", "2", "3"):
        o = outs[flag]
        assert np.array_equal(o.values.view(np.uint64), base.values.view(np.uint64)), (kind, variant, flag)
        assert np.array_equal(o.jump_count, base.jump_count)
        assert np.array_equal(o.stats, base.stats)
        assert np.array_equal(o.sum.view(np.uint64), base.sum.view(np.uint64))
    ref = oracle_lib.run(pk, seed, 0, n, max_jumps=64)
    assert ref["rc"] == 0
    np.testing.assert_array_equal(base.jump_count, ref["jump_count"])
    np.testing.assert_allclose(base.values, ref["values"], rtol=0, atol=1e-6)
