"""Load tests/golden/*.npz (made by tests/golden/make_golden.py from the
reference) into this package's problem types plus the reference outputs."""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from paper_1810_03047_b200.csr import CsrMatrix
from paper_1810_03047_b200.problem import OdeConfig, QuantumProblem, RunOptions
from paper_1810_03047_b200.qops import EffectiveGenerator

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SEED = 987654321


@dataclass
class Sample:
    kind: str
    traj: np.ndarray
    values: np.ndarray
    jump_count: np.ndarray
    jump_t: list
    jump_idx: list
    n_draws: np.ndarray
    psi_points: np.ndarray
    psi: np.ndarray


@dataclass
class Golden:
    name: str
    problem: QuantumProblem
    h0: float
    samples: dict
    raw: dict


def _csr(z, prefix, n):
    return CsrMatrix(n, z[f"{prefix}_row_ptr"], z[f"{prefix}_col_ind"], z[f"{prefix}_values"])


def load(name: str) -> Golden:
    z = dict(np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"), allow_pickle=False))
    n = int(z["prob_dim"])
    init = float(z["prob_initial_step"])
    method = str(z["prob_method"]) if "prob_method" in z else "adams"
    ode = OdeConfig(method=method, rtol=float(z["prob_rtol"]), atol=float(z["prob_atol"]),
                    max_order=int(z["prob_max_order"]), max_steps=int(z["prob_max_steps"]),
                    initial_step=None if np.isnan(init) else init)
    g0 = CsrMatrix(n, z["prob_g_row_ptr"], z["prob_g_col_ind"], z["prob_g_values"])
    gen, rhs = EffectiveGenerator(g0), None
    if "prob_n_td" in z:  # time-dependent right side (timedep.py)
        from paper_1810_03047_b200.timedep import Coefficient, TimeDependentGenerator
        coef = z["prob_td_coef"].reshape(-1, 4)
        rhs = TimeDependentGenerator(g0, [(_csr(z, f"prob_td{k}", n), Coefficient(*map(float, coef[k])))
                                          for k in range(int(z["prob_n_td"]))])
        gen = None
    p = QuantumProblem(
        generator=gen, rhs_fn=rhs,
        collapse_csr=tuple(_csr(z, f"prob_c{i}", n) for i in range(int(z["prob_n_collapse"]))),
        expect_csr=tuple(_csr(z, f"prob_e{i}", n) for i in range(int(z["prob_n_expect"]))),
        psi0=z["prob_psi0"], t_from=float(z["prob_t_from"]), t_to=float(z["prob_t_to"]),
        n_steps=int(z["prob_n_steps"]), ode=ode, options=RunOptions(log_jumps=True))
    samples = {}
    for kind in [str(k) for k in z.get("kinds", [])]:
        counts = z[f"{kind}_jump_count"]
        offs = np.concatenate([[0], np.cumsum(counts)])
        jt = [z[f"{kind}_jump_t"][offs[i]:offs[i + 1]] for i in range(len(counts))]
        ji = [z[f"{kind}_jump_idx"][offs[i]:offs[i + 1]] for i in range(len(counts))]
        samples[kind] = Sample(kind, z[f"{kind}_traj"], z[f"{kind}_values"], counts, jt, ji,
                               z[f"{kind}_n_draws"], z[f"{kind}_psi_points"], z[f"{kind}_psi"])
    return Golden(name, p, float(z["prob_h0"]), samples, z)


CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5")
SCENARIOS = ("decay_forced_jump", "decay_no_jump", "decay_streams", "rabi_closed",
             "rabi_collapse", "photon", "unitary", "trilinear")

TD_NAMES = ("td_rabi", "td_cavity", "td_ising")
BDF_NAMES = ("bdf_c1", "bdf_c2", "bdf_c3", "bdf_stiff", "bdf_decay_forced_jump")

SCRIPTS = {"decay_forced_jump": [[0.5, 0.3, 0.9999999]],
           "bdf_decay_forced_jump": [[0.5, 0.3, 0.9999999]],
           "decay_no_jump": [[float(np.exp(-1.0) / 2)]]}


@dataclass
class Scale:
    """BASELINE-scale reference outputs (tests/golden/scale_<cN>.npz, made by
    make_scale_golden.py from the reference itself)."""
    name: str
    samples: dict          # kind -> Sample (+ .status per trajectory)
    status: dict           # kind -> [n] ISTATE of an OdeFailure (0 = completed)
    n_psi: int
    farm: dict             # the reference's own run_local_farm ensemble
    raw: dict


def load_scale(name: str) -> Scale:
    z = dict(np.load(os.path.join(GOLDEN_DIR, f"scale_{name}.npz"), allow_pickle=False))
    samples, status = {}, {}
    for kind in ("philox", "lfsr113"):
        counts = z[f"{kind}_jump_count"]
        offs = np.concatenate([[0], np.cumsum(counts)])
        jt = [z[f"{kind}_jump_t"][offs[i]:offs[i + 1]] for i in range(len(counts))]
        ji = [z[f"{kind}_jump_idx"][offs[i]:offs[i + 1]] for i in range(len(counts))]
        samples[kind] = Sample(kind, z[f"{kind}_traj"], z[f"{kind}_values"], counts, jt, ji,
                               1 + 2 * counts, z[f"{kind}_psi_points"], z[f"{kind}_psi"])
        status[kind] = z[f"{kind}_status"]
    farm = {k[5:]: z[k] for k in z if k.startswith("farm_")}
    return Scale(name, samples, status, int(z["philox_n_psi"]), farm, z)
