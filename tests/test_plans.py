"""The reference's per-colour index plans (smoothers.py:25-34, 42-118):
compile_plan / PlanBundle return {"red": ColourPlan, "black": ColourPlan}
equal, array for array, to the reference's -- against golden fixtures made
by the reference (tests/golden/make_plans_golden.py) and, where the
reference is importable, against it directly on larger grids."""

import os
import sys

import numpy as np
import pytest

from paper_2110_08389_b200 import smoothers

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from plan_codec import SCHEMES, SIZES, flatten_plans  # noqa: E402

GOLD = np.load(os.path.join(HERE, "golden", "plans.npz"))


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("nx,ny", SIZES)
def test_plans_match_reference_golden(scheme, nx, ny):
    ours = flatten_plans(f"{scheme}_{nx}x{ny}", smoothers.compile_plan(scheme, nx, ny))
    for key, val in ours.items():
        assert np.array_equal(val, GOLD[key]), key


def test_plan_object_shape():
    plans = smoothers.PlanBundle(12, 10).plans("tweed")
    assert set(plans) == {"red", "black"}
    p = plans["black"]
    assert isinstance(p, smoothers.ColourPlan)
    ii, jj, offs, bi, bj = p.legged[0]
    assert ii.dtype == np.int64 and jj.dtype == np.int64 and offs.dtype == np.int64
    assert isinstance(bi, int) and isinstance(bj, int)
    assert offs[0] == 0 and offs[-1] == len(ii)
    assert plans["red"].points_i.dtype == np.int64
    b = smoothers.PlanBundle(8, 8)
    assert b.plans("wireframe") is b.plans("wireframe")  # cached


def test_plan_errors():
    with pytest.raises(ValueError):
        smoothers.compile_plan("plaid", 8, 8)
    with pytest.raises(ValueError):
        smoothers.compile_plan("tweed", 7, 8)
    with pytest.raises(ValueError):
        smoothers.compile_plan("wireframe", 2, 8)


@pytest.mark.parametrize("scheme", ["tweed", "wireframe", "zebra_y"])
@pytest.mark.parametrize("nx,ny", [(64, 48), (48, 90), (130, 130)])
def test_plans_match_live_reference(ref, scheme, nx, ny):
    a = flatten_plans("t", smoothers.compile_plan(scheme, nx, ny))
    b = flatten_plans("t", ref.smoothers.compile_plan(scheme, nx, ny))
    assert a.keys() == b.keys()
    for key in a:
        assert np.array_equal(a[key], b[key]), key
