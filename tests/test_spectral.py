"""Two-grid analyser (spectral.py:1-120) against the
reference's own results (tests/golden/spectral.npz, make_spectral_golden.py):
the small dense-oracle configurations of the reference suite, the pre/post
split at n = 16 and the paper-scale (n = 128) table configurations."""

import os

import numpy as np
import pytest

from paper_2110_08389_b200 import grid

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "spectral.npz"))
SMALL = [("checkerboard", "full", 1, 0), ("zebra_x", "full", 1, 0),
         ("zebra_alt", "full", 1, 0), ("tweed", "full", 1, 0),
         ("tweed", "full", 1, 1), ("wireframe", "half", 1, 0),
         ("tweed_wire_alt", "full", 2, 0), ("zebra_y", "half", 1, 1)]
SPLIT = [(2, 0), (1, 1), (0, 2)]
PAPER = [("uniform", None, "checkerboard", "full", 1), ("uniform", None, "checkerboard", "half", 1),
         ("uniform", None, "tweed", "full", 3), ("wall", 1.5, "tweed", "full", 2),
         ("wall", 1.5, "zebra_alt", "full", 1), ("wall", 3.0, "tweed", "full", 1),
         ("wall", 3.0, "zebra_alt", "full", 2), ("centre", 1.5, "wireframe", "full", 2),
         ("centre", 1.5, "zebra_alt", "full", 1)]


def _pair(kind, n, c):
    x = grid.make_coords(kind, n, 1.0, c)
    return grid.Level(x, x), grid.Level(grid.coarsen(x), grid.coarsen(x))


def _same(res, ref, rtol, dit):
    rho, conv, osc, iters = ref
    assert abs(res[0] - rho) <= rtol * max(rho, 1e-300)
    assert bool(res[1]) == bool(conv) and bool(res[2]) == bool(osc)
    assert abs(res[3] - iters) <= dit


# -- CPU: the oracle's restatement pinned to the reference's results --------

@pytest.mark.parametrize("k", range(len(SMALL)))
def test_oracle_two_grid_small(orc, k):
    sm, rs, n1, n2 = SMALL[k]
    x = grid.make_coords("wall", 8, 1.0, 2.0).values
    got = orc.two_grid_apply(x, x, GOLD["probe"], sm, rs, n1, n2)
    ref = GOLD[f"small_{k}_apply"]
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    _same(orc.spectral_radius(x, x, sm, rs, n1, n2), GOLD[f"small_{k}"], 1e-9, 1)


def test_oracle_split_invariance(orc):
    x = grid.make_coords("centre", 16, 1.0, 1.5).values
    for k, (n1, n2) in enumerate(SPLIT):
        _same(orc.spectral_radius(x, x, "wireframe", "full", n1, n2), GOLD[f"split_{k}"], 1e-9, 1)


# -- GPU: the device analyser -------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(SMALL)))
def test_two_grid_small(cuda, k):
    from paper_2110_08389_b200 import spectral
    sm, rs, n1, n2 = SMALL[k]
    fine, coarse = _pair("wall", 8, 2.0)
    cfg = spectral.TwoGridConfig(fine, coarse, smoother=sm, restriction=rs, nu1=n1, nu2=n2)
    ref = GOLD[f"small_{k}_apply"]
    got = spectral.two_grid_apply(cfg, GOLD["probe"])
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    r = spectral.spectral_radius(cfg)
    _same((r.rho, r.converged, r.oscillation, r.iters), GOLD[f"small_{k}"], 1e-8, 2)


@pytest.mark.gpu
def test_two_grid_zero_and_determinism(cuda):
    from paper_2110_08389_b200 import spectral
    fine, coarse = _pair("wall", 8, 2.0)
    cfg = spectral.TwoGridConfig(fine, coarse)
    assert np.all(spectral.two_grid_apply(cfg, np.zeros(49)) == 0.0)
    cfg2 = spectral.TwoGridConfig(fine, coarse, smoother="tweed", nu1=2)
    a, b = spectral.spectral_radius(cfg2), spectral.spectral_radius(cfg2)
    assert a.rho == b.rho and a.iters == b.iters
    with pytest.raises(ValueError):
        spectral.TwoGridConfig(fine, coarse, nu1=0, nu2=0)
    with pytest.raises(ValueError):
        spectral.TwoGridConfig(fine, fine)


@pytest.mark.gpu
def test_split_invariance(cuda):
    from paper_2110_08389_b200 import spectral
    fine, coarse = _pair("centre", 16, 1.5)
    for k, (n1, n2) in enumerate(SPLIT):
        cfg = spectral.TwoGridConfig(fine, coarse, smoother="wireframe", nu1=n1, nu2=n2)
        r = spectral.spectral_radius(cfg)
        _same((r.rho, r.converged, r.oscillation, r.iters), GOLD[f"split_{k}"], 1e-8, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(PAPER)))
def test_paper_scale_tables(cuda, k):
    """n = 128 (coarse interior 63^2 solved with the device dense inverse)."""
    from paper_2110_08389_b200 import spectral
    kind, c, sm, rs, nu = PAPER[k]
    fine, coarse = _pair(kind, 128, c)
    cfg = spectral.TwoGridConfig(fine, coarse, smoother=sm, restriction=rs, nu1=nu, nu2=0)
    r = spectral.spectral_radius(cfg)
    _same((r.rho, r.converged, r.oscillation, r.iters), GOLD[f"paper_{k}"], 1e-6, 5)
