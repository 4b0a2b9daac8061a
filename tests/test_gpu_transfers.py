"""The V-cycle's residual + restriction on the hybrid session layout
(restrict2_kernel, csrc/tmg_transfer.cu) against the CPU oracle's defect and restriction
(stencil.py:91-96, transfer.py:21-39, mgcycle.py:98-100): bit for bit, for
the tweed, wireframe and zebra_x layouts, full and half weighting, square and
rectangular grids, sizes that are and are not multiples of the 64-point
tiles."""

import ctypes

import numpy as np
import pytest

from paper_2110_08389_b200 import _lib, grid
from paper_2110_08389_b200.rng import Lcg64

pytestmark = pytest.mark.gpu

CASES = [("tweed", 256, 256), ("tweed", 512, 512), ("tweed", 1030, 770), ("tweed", 2048, 2048),
         ("wireframe", 512, 512), ("wireframe", 770, 1030), ("zebra_x", 512, 386),
         ("tweed", 130, 130)]


@pytest.mark.parametrize("kind,nx,ny", CASES)
@pytest.mark.parametrize("full", [1, 0])
def test_session_restriction_bit_exact(cuda, orc, kind, nx, ny, full):
    x = grid.make_coords("wall", nx, 1.0, 3.0)
    y = grid.make_coords("centre", ny, 1.0, 1.5)
    h = grid.build_hierarchy(x, y)
    rng = Lcg64(21 + nx)
    f = np.zeros((nx + 1, ny + 1))
    f[1:-1, 1:-1] = rng.fill((nx - 1, ny - 1)) - 0.5
    u = rng.fill((nx + 1, ny + 1)) - 0.5  # boundary values too
    L = _lib.lib()
    s = ctypes.c_void_p(cuda.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    ud, fd = cuda.from_numpy(u).cuda(), cuda.from_numpy(f).cuda()
    hn = h.native()
    _lib.check(L.tmg_session_load(hn, _lib.KIND_IDS[kind], P(ud), P(fd), s))
    _lib.check(L.tmg_session_restrict(hn, 0, full, s))
    nxc, nyc = nx // 2, ny // 2
    fc = cuda.empty((nxc + 1, nyc + 1), dtype=cuda.float64, device="cuda")
    uc = cuda.empty_like(fc)
    _lib.check(L.tmg_session_read(hn, 1, 1, P(fc), s))
    _lib.check(L.tmg_session_read(hn, 1, 0, P(uc), s))
    st = h.finest.stencil
    d = orc.defect((st.W, st.E, st.S, st.N), u, f)
    want = orc.restrict("full" if full else "half", d)
    got = fc.cpu().numpy()
    assert np.array_equal(got[1:-1, 1:-1], want[1:-1, 1:-1])
    assert not uc.cpu().numpy()[1:-1, 1:-1].any()
