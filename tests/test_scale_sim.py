"""The scheduling model behind DESIGN.md §5 (tools/scale_sim.py): closed-form cases."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import scale_sim  # noqa: E402


def test_one_wave_ends_with_the_longest_trajectory():
    work = np.array([3.0, 5.0, 2.0, 7.0])
    # 4 SMs x 1 CTA: every trajectory alone on its SM
    assert abs(scale_sim.simulate([work], 4, 1, 2.0, 3.0) - 14.0) < 1e-9


def test_pairs_share_an_sm_until_one_finishes():
    # one SM, two CTAs, works 2 and 6: both at tau2 = 3 until the first ends (t = 6),
    # the second then runs its remaining 4 units alone at tau1 = 2: t = 14
    assert abs(scale_sim.simulate([np.array([2.0, 6.0])], 1, 2, 2.0, 3.0) - 14.0) < 1e-9


def test_equal_work_fills_waves_and_a_shared_queue_changes_nothing():
    work = np.full(16, 10.0)
    # 2 SMs x 2 CTAs = 4 slots, 16 equal trajectories: 4 full waves at tau2
    t = scale_sim.simulate([work], 2, 2, 1.0, 1.5)
    assert abs(t - 4 * 10.0 * 1.5) < 1e-9
    # two GPUs: static halves and one global queue take the same time
    static = scale_sim.simulate([work[:8], work[8:]], 2, 2, 1.0, 1.5)
    shared = scale_sim.simulate(2, 2, 2, 1.0, 1.5, shared_queue=work)
    assert abs(static - 2 * 10.0 * 1.5) < 1e-9 and abs(shared - static) < 1e-9


def test_longest_first_never_loses_to_index_order_on_a_tail():
    rng = np.random.default_rng(5)
    work = rng.gamma(40.0, 17.0, 512)
    idx = scale_sim.simulate([work], 148, 2, 9.4e-6, 12.2e-6)
    lpt = scale_sim.simulate([np.sort(work)[::-1]], 148, 2, 9.4e-6, 12.2e-6)
    assert lpt <= idx * (1 + 1e-12)
