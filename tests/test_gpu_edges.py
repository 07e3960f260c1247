"""Edge cases of the device path: empty trajectory ranges, problems without
observables, dimensions that are not a multiple of a warp, and states larger
than every shared-memory staging (d = 3000, CSR from L2, history rows in the
overflow scratch) -- each against the C oracle on identical streams."""

import numpy as np
import pytest

from paper_1810_03047_b200.csr import CsrMatrix
from paper_1810_03047_b200.engine import DeviceProblem, run_gpu
from paper_1810_03047_b200.packing import pack_problem
from paper_1810_03047_b200.problem import OdeConfig, QuantumProblem, RunOptions
from paper_1810_03047_b200.qops import EffectiveGenerator, OperatorSet, coherent, destroy, fock

pytestmark = pytest.mark.gpu

SEED = 987654321
TOL = 1e-6


def _check(pk, n, oracle_lib, **kw):
    with DeviceProblem(pk, **kw) as dp:
        out = dp.run(SEED, 0, n, max_jumps=64)
    ref = oracle_lib.run(pk, SEED, 0, n, max_jumps=64)
    assert out.rc == ref["rc"] == 0, (out.error, ref["error"])
    np.testing.assert_array_equal(out.jump_count, ref["jump_count"])
    for i in range(n):
        m = int(ref["jump_count"][i])
        np.testing.assert_array_equal(out.jump_idx[i, :m], ref["jump_idx"][i, :m])
        np.testing.assert_allclose(out.jump_t[i, :m], ref["jump_t"][i, :m], rtol=0, atol=TOL)
    np.testing.assert_allclose(out.values, ref["values"], rtol=0, atol=TOL)
    return out


def _cavity(n_fock, expect=True, t_to=5.0, n_steps=50):
    a = destroy(n_fock)
    ad = a.conj().T
    ops = OperatorSet(0.4 * (ad @ a) + 0.8 * (a + ad), (np.sqrt(0.3) * a,),
                      (ad @ a, (a + ad) / 2) if expect else ())
    return QuantumProblem.from_operators(ops, coherent(n_fock, 1.5), 0.0, t_to, n_steps,
                                         ode=OdeConfig(rtol=1e-8, atol=1e-10),
                                         options=RunOptions(log_jumps=True))


def test_empty_trajectory_range():
    pk = pack_problem(_cavity(12))
    with DeviceProblem(pk) as dp:
        out = dp.run(SEED, 7, 7)
    assert out.rc == 0 and out.n_failed == 0
    assert np.all(out.sum == 0.0)


def test_no_observables(oracle_lib):
    p = _cavity(12, expect=False)
    res = run_gpu(p, 64, SEED)
    assert res.values.shape == (0, p.n_steps + 1) and res.n_trajectories == 64
    # the jump process itself still matches the oracle
    _check(pack_problem(p), 64, oracle_lib)


@pytest.mark.parametrize("n_fock", [37, 61, 130])
def test_ragged_dimensions(n_fock, oracle_lib):
    _check(pack_problem(_cavity(n_fock)), 32, oracle_lib)


def test_dimension_3000(oracle_lib):
    """A 3000-level driven damped oscillator: past every shared-memory
    staging (G read as CSR through L1/L2, two history rows in registers,
    the rest in the overflow scratch)."""
    import scipy.sparse as sp
    dim = 3000

    def csr(m):
        m = sp.csr_matrix(m, dtype=np.complex128)
        m.eliminate_zeros()
        m.sort_indices()
        return CsrMatrix(dim, m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data)
    a = sp.diags(np.sqrt(np.arange(1, dim, dtype=np.float64)), 1, format="csr")
    ad = a.T.tocsr()
    n = ad @ a
    h = 0.4 * n + 0.8 * (a + ad)
    c = np.sqrt(0.3) * a
    g = -1j * h - 0.5 * (c.T @ c)
    p = QuantumProblem(generator=EffectiveGenerator(csr(g)), collapse_csr=(csr(c),),
                       expect_csr=(csr(n), csr((a + ad) / 2)), psi0=fock(dim, 3),
                       t_from=0.0, t_to=3.0, n_steps=30, ode=OdeConfig(rtol=1e-8, atol=1e-10),
                       options=RunOptions(log_jumps=True))
    pk = pack_problem(p)
    _check(pk, 8, oracle_lib)


@pytest.mark.parametrize("n_fock", [3, 4])
def test_small_kernel_three_and_four_levels(n_fock, oracle_lib):
    """d = 3 and 4 run on the one-thread-per-trajectory kernel with d_max = 4
    (variant 42, automatic for 2 < d <= 4): padded components inactive."""
    pk = pack_problem(_cavity(n_fock))
    out = _check(pk, 96, oracle_lib)
    assert out.variant == 42


@pytest.mark.parametrize("n_fock", [600, 777])
def test_tmem_variant_on_ragged_dimensions(n_fock, oracle_lib):
    """The TMEM history variant (automatic for 512 < d <= 1024) on states
    that fill only part of its 1024 components."""
    out = _check(pack_problem(_cavity(n_fock, t_to=1.0, n_steps=10)), 16, oracle_lib)
    assert out.variant == 39


def test_fp64_pipe_probes():
    """The roofline denominators are measured on the device: DFMA and the
    FP64 tensor pipe (DMMA m8n8k4).  B200's FP64 tensor throughput is no
    higher than its DFMA throughput (why no dense DMMA path)."""
    from paper_1810_03047_b200 import native
    dfma = native.fp64_peak_tflops(0)
    dmma = native.dmma_peak_tflops(0)
    assert 10.0 < dfma < 100.0 and 5.0 < dmma < 200.0
    print(f"DFMA {dfma:.1f} TFLOP/s, DMMA {dmma:.1f} TFLOP/s")


@pytest.mark.parametrize("case", ["c1_small", "c2_smem_hist", "c4_tmem", "c4_regs", "c4td",
                                  "c5_two_cta", "c2_bdf"])
def test_repeat_runs_are_bitwise_identical(case):
    """Every kernel family twice on the same inputs, with different launch
    interleavings (a second problem handle launched in between): per-
    trajectory series, jump logs and counters identical to the bit.  Shared-
    memory, TMEM or scheduling races would show up here as run-to-run
    differences (compute-sanitizer is closed on the GPU pool; this is the
    determinism check that stands in for racecheck)."""
    import dataclasses
    from paper_1810_03047_b200 import configs
    name, _, kind = case.partition("_")
    variant = {"small": 40, "smem_hist": 17, "tmem": 39, "regs": 22, "two_cta": 27}.get(kind, -1)
    p = configs.build(name)
    if kind == "bdf":
        p = dataclasses.replace(p, ode=OdeConfig(method="bdf", rtol=p.ode.rtol, atol=p.ode.atol))
    n = {"c1": 500, "c2": 256, "c4": 300, "c4td": 160, "c5": 96}[name]
    if kind == "bdf":
        n = 32
    with DeviceProblem(p, variant=variant) as dp, DeviceProblem(p, variant=variant) as other:
        a = dp.run(SEED, 0, n, max_jumps=64)
        other.run(SEED + 1, 0, n // 2, max_jumps=64)
        b = dp.run(SEED, 0, n, max_jumps=64)
    assert a.rc == b.rc
    np.testing.assert_array_equal(a.values, b.values)
    np.testing.assert_array_equal(a.jump_count, b.jump_count)
    np.testing.assert_array_equal(a.jump_t, b.jump_t)
    np.testing.assert_array_equal(a.stats, b.stats)
    np.testing.assert_array_equal(a.sum, b.sum)
