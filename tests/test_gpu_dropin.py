"""The drop-in on the device: the reference's own problem objects in, the
reference's own result and exception classes out (run_gpu replaces
mcwf.run_inline, cluster.py:472-482)."""

import dataclasses
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

pytestmark = pytest.mark.gpu

ref_configs = pytest.importorskip("ref_configs")
import mcwf  # noqa: E402

import goldens  # noqa: E402
from paper_1810_03047_b200 import configs, run_gpu  # noqa: E402


def test_run_gpu_on_reference_problem():
    p = ref_configs.c2()
    res = run_gpu(p, 300, goldens.SEED)
    assert isinstance(res, mcwf.TrajectoryResult)
    assert res.n_trajectories == 300 and res.values.shape == (2, 301)
    assert res.jumps is not None  # the reference problem asks for the jump log
    own = run_gpu(configs.build("c2"), 300, goldens.SEED)
    np.testing.assert_array_equal(res.values, own.values)
    assert np.all(np.isfinite(res.standard_error()))


def test_reference_odefailure_is_caught():
    g = goldens.load("c1_max_steps")
    p = dataclasses.replace(ref_configs.c1(),
                            ode=mcwf.OdeConfig(rtol=1e-8, atol=1e-10, max_steps=1))
    with pytest.raises(mcwf.OdeFailure) as exc:
        run_gpu(p, 4, goldens.SEED)
    assert str(exc.value) == str(g.raw["max_steps_msg"])
    assert exc.value.istate == int(g.raw["max_steps_istate"])
