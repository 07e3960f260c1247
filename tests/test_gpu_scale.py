"""Device vs the REFERENCE ITSELF at BASELINE scale.

Fixtures: tests/golden/scale_<cN>.npz, made by tests/golden/make_scale_golden.py
from the reference's own ``run_single_trajectory`` (trajectory.py:190-250)
and its own farm (run_local_farm, cluster.py:493-516).

* Identical streams -- every trajectory of c1 (500) and the first 256 of
  c2-c5, under Philox and under the reference's LFSR113 generator
  (derive_stream(seed, k), rng.py:76-90): OdeFailure status identical,
  jump counts and channels exact, jump times / <O_k>(t_j) / psi(t_j) within
  1e-6 per trajectory, the sample ensemble within 1e-6.  c5 alone is worse
  conditioned than 1e-6 for any implementation that is not bit-identical to
  the reference: its per-trajectory bound is 4x the reference algorithm's
  own one-ulp sensitivity on the same sample, measured here and printed.
* Independent streams -- the device ensemble at the config's full N
  (Philox) against the reference's own ensemble (run_local_farm's
  per-worker sequential LFSR113 streams, cluster.py:415-420): per point
  |delta| <= 3 sqrt(SE_gpu^2 + SE_ref^2) up to the expected tail.
* c4's two reference-faithful failures: OdeFailure(-5) on trajectories 3016
  and 3438 of the 4096-trajectory Philox ensemble, with the reference's
  exception text.
"""

import numpy as np
import pytest

import goldens
from sensitivity import self_sensitivity
from paper_1810_03047_b200 import configs, native
from paper_1810_03047_b200.engine import DeviceProblem, raise_for_status
from paper_1810_03047_b200.packing import pack_problem

pytestmark = pytest.mark.gpu

TOL = 1e-6
MAXJ = 256
# device status -> the ISTATE of the OdeFailure the reference raises
ISTATE = {native.ERR_MAX_STEPS: -1, native.ERR_REPEATED_ERRTEST: -4,
          native.ERR_STEP_COLLAPSE: -5, native.ERR_CORRECTOR: -5, 0: 0}


@pytest.mark.parametrize("name", goldens.CONFIG_NAMES)
@pytest.mark.parametrize("kind", ["philox", "lfsr113"])
def test_identical_streams_vs_reference_at_scale(name, kind, oracle_lib, capsys):
    sc = goldens.load_scale(name)
    s = sc.samples[kind]
    n = len(s.traj)
    pk = pack_problem(configs.build(name))
    with DeviceProblem(pk) as dp:
        out = dp.run(goldens.SEED, 0, n, stream=kind, max_jumps=MAXJ,
                     psi_points=s.psi_points)
    st = np.array([ISTATE[int(c)] for c in out.status])
    np.testing.assert_array_equal(st, sc.status[kind])
    ok = sc.status[kind] == 0
    tol_t = tol_v = tol_m = TOL
    if name == "c5":
        _, sens_t, sens_v, sens_m = self_sensitivity(oracle_lib, pk, n, stream=kind)
        tol_t, tol_v, tol_m = (max(TOL, 4 * x) for x in (sens_t, sens_v, sens_m))
        with capsys.disabled():
            print(f"\n[c5 {kind}, {n} trajectories] reference one-ulp sensitivity: "
                  f"jump times {sens_t:.2e}, values {sens_v:.2e}, mean {sens_m:.2e} -> "
                  f"per-trajectory bounds {tol_t:.2e} (t*), {tol_v:.2e} (values), "
                  f"ensemble {tol_m:.2e}")
    worst_t = worst_v = 0.0
    for i in np.nonzero(ok)[0]:
        m = int(s.jump_count[i])
        assert int(out.jump_count[i]) == m, i
        np.testing.assert_array_equal(out.jump_idx[i, :m], s.jump_idx[i])
        if m:
            worst_t = max(worst_t, float(np.abs(out.jump_t[i, :m] - s.jump_t[i]).max()))
        worst_v = max(worst_v, float(np.abs(out.values[i] - s.values[i]).max()))
    dmean = float(np.abs(out.values[ok].mean(axis=0) - s.values[ok].mean(axis=0)).max())
    with capsys.disabled():
        print(f"\n[{name} {kind}, {n} trajectories, {int((~ok).sum())} reference failures] "
              f"device vs reference: max |dt*| {worst_t:.2e}, max |dvalue| {worst_v:.2e}, "
              f"max |dmean| {dmean:.2e}")
    assert worst_t <= tol_t, worst_t
    assert worst_v <= tol_v, worst_v
    # psi(t_j) itself for the first trajectories (north_star "psi(t) within 1e-6")
    n_psi = sc.n_psi
    keep = ok[:n_psi]
    np.testing.assert_allclose(out.psi[:n_psi][keep], s.psi[keep], rtol=0, atol=tol_v)
    # ensemble over the sample under identical streams
    np.testing.assert_allclose(out.values[ok].mean(axis=0), s.values[ok].mean(axis=0),
                               rtol=0, atol=tol_m)
    np.testing.assert_array_equal(out.stats[ok, native.STAT_NAMES.index("draws")],
                                  s.n_draws[ok])


@pytest.mark.parametrize("name", goldens.CONFIG_NAMES)
def test_independent_streams_vs_reference_farm(name):
    """Full-N device ensemble vs the reference's own run_local_farm ensemble
    (c1 500, c2 5000, c3 2000, c4 4096, c5 256 trajectories on 8 workers)."""
    sc = goldens.load_scale(name)
    f = sc.farm
    n_ref = int(f["n"])
    mc = f["sum"] / n_ref
    np.testing.assert_allclose(mc, f["mean"], rtol=0, atol=1e-12)  # the farm's own average
    var_c = np.maximum(f["sumsq"] / n_ref - mc ** 2, 0) * n_ref / (n_ref - 1)
    p = configs.build(name)
    n_gpu = configs.N_TRAJECTORIES[name]
    with DeviceProblem(p) as dp:
        out = dp.run(goldens.SEED, 0, n_gpu, per_trajectory=False, resident=True)
    n_ok = n_gpu - out.n_failed  # c4: the reference controller's own two collapses
    mg = out.sum / n_ok
    var_g = np.maximum(out.sumsq / n_ok - mg ** 2, 0) * n_ok / (n_ok - 1)
    # a small reference sample (c5: 256) may have no jump yet at early times
    # (sample variance 0); the population variance then comes from the device
    se = np.sqrt(var_g / n_ok + np.maximum(var_c, var_g) / n_ref)
    live = se > 1e-9
    z = np.abs(mg - mc)[live] / se[live]
    # the expected ~0.3 % beyond 3 sigma (plus finite-sample slack), none beyond 5
    assert np.mean(z > 3) < 0.02 and z.max() < 5, (np.mean(z > 3), z.max())


def test_c4_reference_failures():
    """Trajectories 3016 and 3438 of the c4 Philox ensemble make the
    reference's Adams controller collapse (OdeFailure -5, a reject/accept
    limit cycle driving h to ~1e-16); the device raises the same ISTATE with
    the reference's message text (numbers to the printed precision)."""
    sc = goldens.load_scale("c4")
    z = sc.raw
    with DeviceProblem(configs.build("c4")) as dp:
        for k, istate, msg in zip(z["fail_traj"], z["fail_status"], z["fail_msg"]):
            out = dp.run(goldens.SEED, int(k), int(k) + 1, max_jumps=MAXJ)
            assert ISTATE[int(out.status[0])] == int(istate)
            with pytest.raises(RuntimeError) as exc:
                raise_for_status(out.rc, out.error)
            got, want = str(exc.value), str(msg)
            assert got.split(" (step size")[0] == want.split(" (step size")[0]
            # "step size collapsed to <h> at t = <t>": t to the printed digits
            assert got.split("at t = ")[1][:5] == want.split("at t = ")[1][:5]
