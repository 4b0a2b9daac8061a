"""The V-cycle's hybrid N/T field layout (csrc/tmg_layout.h) against the
natural C-order path: conversions round-trip bit-exactly, the residual norm is
bit-identical, sweeps and V-cycles agree to rounding."""

import ctypes
import os

import numpy as np
import pytest

from paper_2110_08389_b200 import _lib, grid, mgcycle
from paper_2110_08389_b200.rng import Lcg64
from paper_2110_08389_b200.stencil import defect_norm, native_level

pytestmark = pytest.mark.gpu

CASES = [("tweed", "wall", 3.0, 64, 64), ("tweed", "wall", 2.0, 64, 40),
         ("tweed", "wall", 2.0, 40, 64), ("wireframe", "centre", 1.5, 64, 64),
         ("wireframe", "centre", 1.5, 72, 48), ("wireframe", "centre", 1.5, 48, 72),
         ("zebra_x", "wall", 2.0, 48, 32)]


def _setup(cuda, kind, stretch, c, n, m, seed=3):
    x = grid.make_coords(stretch, n, 1.0, c)
    y = grid.make_coords(stretch, m, 1.0, c)
    h = grid.build_hierarchy(x, y)
    rng = Lcg64(seed)
    f = np.zeros((n + 1, m + 1))
    f[1:-1, 1:-1] = rng.fill((n - 1, m - 1)) - 0.5
    u = np.zeros_like(f)
    u[1:-1, 1:-1] = rng.fill((n - 1, m - 1)) - 0.5
    u[0, :], u[-1, :], u[:, 0], u[:, -1] = 0.3, -0.2, 0.1, 0.05
    return h, cuda.from_numpy(u).cuda(), cuda.from_numpy(f).cuda()


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _s(cuda):
    return ctypes.c_void_p(cuda.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("kind,stretch,c,n,m", CASES)
def test_session_roundtrip_and_norm(cuda, kind, stretch, c, n, m):
    h, u, f = _setup(cuda, kind, stretch, c, n, m)
    L = _lib.lib()
    hn = h.native()
    k = _lib.KIND_IDS[kind]
    _lib.check(L.tmg_session_load(hn, k, _p(u), _p(f), _s(cuda)))
    out = cuda.full_like(u, 7.0)
    _lib.check(L.tmg_session_store(hn, _p(out), _s(cuda)))
    assert cuda.equal(out, u)
    v = ctypes.c_double()
    _lib.check(L.tmg_session_norm(hn, ctypes.byref(v), _s(cuda)))
    assert v.value == defect_norm(h.finest.stencil, u, f)


@pytest.mark.parametrize("kind,stretch,c,n,m", CASES)
def test_session_sweeps_match_natural(cuda, kind, stretch, c, n, m):
    h, u, f = _setup(cuda, kind, stretch, c, n, m)
    L = _lib.lib()
    hn = h.native()
    k = _lib.KIND_IDS[kind]
    ref = u.clone()
    lv = native_level(h.finest.stencil)
    for _ in range(2):
        _lib.check(L.tmg_sweep(lv, k, _p(ref), _p(f), _s(cuda)))
    _lib.check(L.tmg_session_load(hn, k, _p(u), _p(f), _s(cuda)))
    _lib.check(L.tmg_session_sweeps(hn, k, 2, _s(cuda)))
    got = cuda.empty_like(u)
    _lib.check(L.tmg_session_store(hn, _p(got), _s(cuda)))
    err = float((got - ref).abs().max() / ref.abs().max())
    assert err <= 1e-12, err


@pytest.mark.parametrize("kind,stretch,c,n,m", CASES)
def test_hybrid_vcycle_matches_natural(cuda, kind, stretch, c, n, m):
    h1, u1, f = _setup(cuda, kind, stretch, c, n, m)
    h2 = grid.build_hierarchy(h1.finest.x, h1.finest.y)
    u2 = u1.clone()
    cfg = mgcycle.CycleConfig(smoother=kind)
    old = os.environ.get("TMG_LAYOUT")
    try:
        os.environ["TMG_LAYOUT"] = "natural"
        for _ in range(2):
            mgcycle.v_cycle(h2, cfg, u2, f)
    finally:
        if old is None:
            os.environ.pop("TMG_LAYOUT", None)
        else:
            os.environ["TMG_LAYOUT"] = old
    for _ in range(2):
        mgcycle.v_cycle(h1, cfg, u1, f)
    err = float((u1 - u2).abs().max() / u2.abs().max())
    assert err <= 1e-12, err
