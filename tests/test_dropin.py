"""The drop-in boundary with the reference package itself (CPU part).

A problem built by the reference's own constructors (mcwf, imported from
/root/reference or from the pip copy in baseline/_ref) packs to exactly the
device form of this package's own c1-c5 (same bytes, same digest), and the
result / exception types handed back carry the reference's classes."""

import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

ref_configs = pytest.importorskip("ref_configs")
import mcwf  # noqa: E402

from paper_1810_03047_b200 import configs  # noqa: E402
from paper_1810_03047_b200.packing import pack_problem  # noqa: E402
from paper_1810_03047_b200.problem import OdeFailure, TrajectoryResult, reference_types  # noqa: E402


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_reference_problem_packs_identically(name):
    a = pack_problem(ref_configs.CONFIGS[name]())
    b = pack_problem(configs.build(name))
    assert a.digest == b.digest
    assert a.h0_first == b.h0_first
    for f in ("psi0", "times", "l_table", "tau1", "tau2", "tau3"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    for x, y in zip([a.g, *a.collapse, *a.expect], [b.g, *b.collapse, *b.expect]):
        np.testing.assert_array_equal(x.row_ptr, y.row_ptr)
        np.testing.assert_array_equal(x.col_ind, y.col_ind)
        np.testing.assert_array_equal(x.values, y.values)


def test_boundary_types_are_the_references():
    fail, res = reference_types(ref_configs.c1())
    assert issubclass(fail, mcwf.OdeFailure) and issubclass(fail, OdeFailure)
    assert issubclass(res, mcwf.TrajectoryResult) and issubclass(res, TrajectoryResult)
    r = res(np.linspace(0, 1, 3), np.zeros((1, 3)), 2, None, sumsq=np.zeros((1, 3)))
    assert isinstance(r, mcwf.TrajectoryResult) and r.standard_error().shape == (1, 3)
    with pytest.raises(mcwf.OdeFailure) as exc:
        raise fail(-5, "x")
    assert exc.value.istate == -5
    assert str(exc.value) == str(mcwf.OdeFailure(-5, "x"))


def test_reference_failure_raised_through_boundary():
    from paper_1810_03047_b200 import native
    from paper_1810_03047_b200.engine import raise_for_status
    with pytest.raises(mcwf.OdeFailure) as exc:
        raise_for_status(native.ERR_MAX_STEPS, {"t": 0.5, "h": 0.1, "max_steps": 1},
                         ref_configs.c1())
    assert exc.value.istate == -1 and str(exc.value).endswith("(inside trajectory))")
