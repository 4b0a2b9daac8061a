"""The reference's own sub-sweep pattern (pkg/tests/test_smoothers.py:27-39,
test_acceptance.py:166-177): walk bundle.plans(kind)[colour] and call the
active kernel module's per-block entry points (kernels.relax_*, the C-ABI
shims of _ckernels.pyx:42-185).  Per colour stage the result equals the CPU
oracle's colour stage, for numpy and CUDA-tensor fields."""

import numpy as np
import pytest

from paper_2110_08389_b200 import grid, kernels, smoothers, stencil
from paper_2110_08389_b200.rng import Lcg64

pytestmark = pytest.mark.gpu


def _sub_sweep(kind, st, bundle, u, f, colour):
    p = bundle.plans(kind)[colour]
    k = kernels.active()
    W, E, S, N = st.W, st.E, st.S, st.N
    if p.points_i.size:
        k.relax_points(p.points_i, p.points_j, W, E, S, N, u, f)
    for ii, jj, offs, bi, bj in p.legged:
        k.relax_legged(ii, jj, offs, bi, bj, W, E, S, N, u, f)
    for ii, jj in p.chains:
        k.relax_chain(ii, jj, W, E, S, N, u, f)
    for ii, jj in p.rings:
        k.relax_ring(ii, jj, W, E, S, N, u, f)


def _setup(nx, ny, seed=13):
    x = grid.make_coords("wall", nx, 1.0, 2.5)
    y = grid.make_coords("wall", ny, 1.0, 1.5)
    st = stencil.assemble(x, y)
    rng = Lcg64(seed)
    f = np.zeros((nx + 1, ny + 1))
    f[1:-1, 1:-1] = rng.fill((nx - 1, ny - 1)) - 0.5
    u = np.zeros_like(f)
    u[1:-1, 1:-1] = rng.fill((nx - 1, ny - 1)) - 0.5
    u[0, :], u[-1, :] = 0.25, -0.125
    return st, u, f


@pytest.mark.parametrize("kind", ["tweed", "wireframe", "zebra_x", "zebra_y", "checkerboard"])
@pytest.mark.parametrize("nx,ny", [(12, 10), (16, 16), (10, 20)])
@pytest.mark.parametrize("on_device", [False, True])
def test_reference_sub_sweep_pattern(cuda, orc, kind, nx, ny, on_device):
    st, u0, f = _setup(nx, ny)
    bundle = smoothers.PlanBundle(nx, ny)
    coefs = (st.W, st.E, st.S, st.N)
    uo = u0.copy()
    u = cuda.from_numpy(u0.copy()).cuda() if on_device else u0.copy()
    fd = cuda.from_numpy(f).cuda() if on_device else f
    for colour, red in (("red", 1), ("black", 0)):
        _sub_sweep(kind, st, bundle, u, fd, colour)
        orc.sweep_part(kind, coefs, uo, f, red, 0, 1 << 30)
        got = u.cpu().numpy() if on_device else u
        err = np.abs(got - uo).max() / np.abs(uo).max()
        assert err <= 1e-12, (colour, err)
