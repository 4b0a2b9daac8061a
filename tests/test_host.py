"""Host-side pieces that need no GPU: the C ABI loads and exports every
declared symbol, the native closed-form geometry equals the oracle's (and the
reference's) layouts, the vectorised LCG equals the scalar recurrence, and
the host setup (grid, assemble) is bit-identical to the reference."""

import os
import re

import numpy as np
import pytest

from paper_2110_08389_b200 import _lib, grid, layout, mgcycle, smoothers, stencil
from paper_2110_08389_b200.rng import INC, MULT, Lcg64

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "tweedmg_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:const char\*|int|long long|long)\s+\**(tmg_\w+)\(",
                              hdr, re.M))
    assert len(declared) >= 25
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert set(_lib.exported_symbols()) == declared
    assert L.tmg_version() >= 100


def test_layout_geometry_matches_oracle(orc):
    for nx in range(4, 31, 2):
        for ny in range(4, 31, 2):
            for kind in ("tweed", "wireframe"):
                ii, jj, bb, fl = layout.member_arrays(kind, nx, ny)
                oi, oj, ob, orr = orc.layout_dump(kind, nx, ny)
                assert np.array_equal(ii, oi) and np.array_equal(jj, oj)
                assert np.array_equal(bb, ob) and np.array_equal(fl & 1, orr)


def test_layout_matches_reference(ref):
    import dataclasses
    for nx in range(4, 41, 2):
        for ny in range(4, 41, 2):
            for fn in ("tweed_layout", "wireframe_layout"):
                a = getattr(layout, fn)(nx, ny)
                b = getattr(ref.layout, fn)(nx, ny)
                assert [dataclasses.astuple(x) for x in a.blocks] == \
                       [dataclasses.astuple(y) for y in b.blocks]


def test_layout_large_grid_is_fast_and_a_partition():
    ii, jj, bb, fl = layout.member_arrays("tweed", 2048, 2048)
    key = ii.astype(np.int64) * 4096 + jj
    assert len(np.unique(key)) == 2047 * 2047


def test_layout_census():
    lay = layout.tweed_layout(6, 6)
    assert sorted(b.kind for b in lay.blocks) == ["legged"] * 5 + ["point"] * 4
    lay = layout.tweed_layout(8, 6)
    assert len([b for b in lay.blocks if b.kind == "legged" and len(b.legs) == 3]) == 2
    rep = layout.edge_cover_check(layout.tweed_layout(12, 10), layout.wireframe_layout(12, 10))
    assert rep.disjoint and rep.covers_all
    with pytest.raises(ValueError):
        layout.tweed_layout(5, 6)


def test_lcg_matches_recurrence():
    mask = (1 << 64) - 1
    state = (12345 ^ INC) & mask
    state = (MULT * state + INC) & mask
    want = []
    for _ in range(9000):
        state = (MULT * state + INC) & mask
        want.append((state >> 11) / float(1 << 53))
    assert Lcg64(12345).fill(9000).tolist() == want
    g = Lcg64(3)
    assert np.array_equal(g.fill((2, 3)).ravel(), Lcg64(3).fill(6))


def test_lcg_matches_reference(ref):
    from tweedmg.rng import Lcg64 as R
    for seed in (0, 1, 2, 99):
        assert np.array_equal(Lcg64(seed).fill(10007), R(seed).fill(10007))


def test_host_setup_matches_reference(ref):
    for kind, c in (("uniform", None), ("wall", 3.0), ("centre", 1.5)):
        for n in (4, 16, 128):
            a = grid.make_coords(kind, n, 1.0, c)
            b = ref.grid.make_coords(kind, n, 1.0, c)
            assert np.array_equal(a.values, b.values)
            sa, sb = stencil.assemble(a, a), ref.stencil.assemble(b, b)
            for p in "WESN":
                assert np.array_equal(getattr(sa, p), getattr(sb, p))
    h = grid.build_hierarchy(grid.make_uniform(128, 1.0), grid.make_uniform(96, 1.0))
    assert [(lv.nx, lv.ny) for lv in h.levels] == [(128, 96), (64, 48), (32, 24), (16, 12),
                                                    (8, 6), (4, 3)]


def test_config_validation():
    with pytest.raises(ValueError):
        mgcycle.CycleConfig(smoother="gingham")
    with pytest.raises(ValueError):
        mgcycle.CycleConfig(nu1=0, nu2=0)
    with pytest.raises(ValueError):
        mgcycle.CycleConfig(tol=0.0)
    assert mgcycle.CycleConfig(smoother="zebra_alt").relaxations_per_cycle == 8
    assert smoothers.sweep_cost("tweed", 5) == 261
    assert smoothers.sweep_cost("wireframe", 5) == 409
    with pytest.raises(ValueError):
        smoothers.compile_plan("plaid", 8, 8)


def test_lcg_jump_ahead_matches_stream():
    from paper_2110_08389_b200.rng import Lcg64
    for seed, n in ((0, 1), (7, 4096), (3, 12345), (11, 5000)):
        a, b = Lcg64(seed), Lcg64(seed)
        a.fill(n)
        b.advance(n)
        assert a.state == b.state


@pytest.mark.gpu
def test_lcg_device_fill_bit_identical(cuda):
    from paper_2110_08389_b200.rng import Lcg64
    for seed, shape in ((0, (7,)), (5, (129, 131)), (2, (1000, 1003))):
        a, b = Lcg64(seed), Lcg64(seed)
        host = a.fill(shape)
        dev = b.fill_device(shape).cpu().numpy()
        assert np.array_equal(host, dev) and a.state == b.state
