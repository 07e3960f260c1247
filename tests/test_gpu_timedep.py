"""Time-dependent H(t) = H0 + sum_k c_k(t) H_k on the device (timedep.py,
the TD kernel variants of csrc/qtm_traj.cuh) vs the reference's general
Adams engine driving the same rhs_fn (golden fixtures) and vs the C oracle
under identical streams.  Same bar as the constant-generator path: jump
sequences exact, series and jump times within 1e-6."""

import numpy as np
import pytest

import goldens
from paper_1810_03047_b200 import native
from paper_1810_03047_b200.engine import DeviceProblem, run_gpu
from paper_1810_03047_b200.packing import pack_problem

pytestmark = pytest.mark.gpu

TOL = 1e-6
MAXJ = 256


def _compare(out, vals, jc, jt, ji, tol=TOL):
    n = len(jc)
    np.testing.assert_array_equal(out.jump_count[:n], jc)
    for i in range(n):
        m = int(jc[i])
        np.testing.assert_array_equal(out.jump_idx[i, :m], ji[i][:m])
        np.testing.assert_allclose(out.jump_t[i, :m], jt[i][:m], rtol=0, atol=tol)
    np.testing.assert_allclose(out.values[:n], vals, rtol=0, atol=tol)


@pytest.mark.parametrize("name", goldens.TD_NAMES)
def test_td_device_matches_reference_goldens(name):
    g = goldens.load(name)
    for kind, s in g.samples.items():
        k0, k1 = int(s.traj[0]), int(s.traj[-1]) + 1
        with DeviceProblem(g.problem) as dp:
            out = dp.run(goldens.SEED, k0, k1, stream=kind, max_jumps=MAXJ, psi_points=s.psi_points)
        assert out.rc == 0, out.error
        assert native.variant_time_dependent(out.variant)
        _compare(out, s.values, s.jump_count, s.jump_t, s.jump_idx)
        np.testing.assert_array_equal(out.stats[:, 11], s.n_draws)
        if len(s.psi_points):  # psi(t_j) within 1e-6 of the reference's recorded states
            np.testing.assert_allclose(out.psi, s.psi, rtol=0, atol=TOL)


@pytest.mark.parametrize("name,n", [("td_rabi", 500), ("td_cavity", 256), ("td_ising", 64)])
def test_td_device_matches_oracle(name, n, oracle_lib):
    pk = pack_problem(goldens.load(name).problem)
    with DeviceProblem(pk) as dp:
        out = dp.run(goldens.SEED, 0, n, max_jumps=MAXJ)
    assert out.rc == 0, out.error
    ref = oracle_lib.run(pk, goldens.SEED, 0, n, max_jumps=MAXJ)
    assert ref["rc"] == 0
    _compare(out, ref["values"], ref["jump_count"], list(ref["jump_t"]), list(ref["jump_idx"]))
    np.testing.assert_allclose(out.sum / n, ref["values"].mean(axis=0), rtol=0, atol=TOL)


def test_td_run_gpu_and_variant_guard(oracle_lib):
    g = goldens.load("td_rabi")
    res = run_gpu(g.problem, 256, goldens.SEED)
    ref = oracle_lib.run(pack_problem(g.problem), goldens.SEED, 0, 256)
    np.testing.assert_allclose(res.values, ref["values"].mean(axis=0), rtol=0, atol=TOL)
    # a constant-generator kernel variant cannot run a time-dependent problem
    plain = next(i for i in range(len(native.variants())) if not native.variant_time_dependent(i))
    with pytest.raises(RuntimeError, match="time-dependent"):
        DeviceProblem(g.problem, variant=plain)


@pytest.mark.parametrize("variant", [-1, 34, 36, 43])
def test_td_c4td_variants_match_oracle(variant, oracle_lib):
    """c4td (bench workload): the automatic TD variant (the TMEM twin, 43: the
    modulated field is a single-valued term, so two CTAs fit an SM), the former
    defaults (512, 2, 8) and (256, 4, 8) in registers, vs the oracle."""
    from paper_1810_03047_b200 import configs
    assert native.variant_time_dependent(36) and native.variant_time_dependent(37)
    assert native.variant_time_dependent(43) and native.variant_tmem_rows(43) > 0
    pk = pack_problem(configs.build("c4td"))
    n = 48
    with DeviceProblem(pk, variant=variant) as dp:
        if variant == -1:
            assert dp.layout()["variant"] == 43 and dp.max_resident() >= 2 * 132  # two CTAs per SM
        out = dp.run(goldens.SEED, 0, n, max_jumps=MAXJ)
    ref = oracle_lib.run(pk, goldens.SEED, 0, n, max_jumps=MAXJ)
    assert out.rc == ref["rc"]
    ok = ref["status"] == 0
    np.testing.assert_array_equal(out.status, ref["status"])
    np.testing.assert_array_equal(out.jump_count[ok], ref["jump_count"][ok])
    np.testing.assert_allclose(out.values[ok], ref["values"][ok], rtol=0, atol=TOL)


@pytest.mark.parametrize("variant", [28, 30, 37])
def test_td_other_variants_match_oracle(variant, oracle_lib):
    pk = pack_problem(goldens.load("td_cavity").problem)
    n = 64
    with DeviceProblem(pk, variant=variant) as dp:
        out = dp.run(goldens.SEED, 0, n, max_jumps=MAXJ)
    assert out.rc == 0, out.error
    ref = oracle_lib.run(pk, goldens.SEED, 0, n, max_jumps=MAXJ)
    _compare(out, ref["values"], ref["jump_count"], list(ref["jump_t"]), list(ref["jump_idx"]))
