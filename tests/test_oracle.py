"""The CPU oracle is pinned to the reference: bit-identical sweeps, residual,
transfers and solves (this container, where the reference is importable)."""

import numpy as np
import pytest


def _setup(ref, stretch, c, nx, ny, seed=31):
    x = ref.grid.make_coords(stretch, nx, 1.0, c)
    y = ref.grid.make_coords(stretch, ny, 1.0, c)
    st = ref.stencil.assemble(x, y)
    from tweedmg.rng import Lcg64
    rng = Lcg64(seed)
    f = np.zeros((nx + 1, ny + 1))
    f[1:-1, 1:-1] = rng.fill((nx - 1, ny - 1)) - 0.5
    u = np.zeros_like(f)
    u[1:-1, 1:-1] = rng.fill((nx - 1, ny - 1)) - 0.5
    return x, y, st, u, f


KINDS = ("checkerboard", "zebra_x", "zebra_y", "zebra_alt", "tweed", "wireframe",
         "tweed_wire_alt")


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("nx,ny", [(12, 10), (10, 10), (8, 14), (20, 8)])
@pytest.mark.parametrize("stretch,c", [("uniform", None), ("wall", 3.0), ("centre", 1.5)])
def test_oracle_sweeps_bit_exact(ref, orc, kind, nx, ny, stretch, c):
    x, y, st, u, f = _setup(ref, stretch, c, nx, ny)
    W, E, S, N = orc.assemble(x.values, y.values)
    for a, b in zip((W, E, S, N), (st.W, st.E, st.S, st.N)):
        assert np.array_equal(a, b)
    bundle = ref.smoothers.PlanBundle(nx, ny)
    uo = u.copy()
    for _ in range(3):
        ref.smoothers.sweep(kind, st, bundle, u, f)
        orc.sweep(kind, (W, E, S, N), uo, f, nthreads=2)
    assert np.array_equal(u, uo)
    d = ref.stencil.defect(st, u, f)
    assert np.array_equal(d, orc.defect((W, E, S, N), u, f))
    for rk in ("half", "full"):
        assert np.array_equal(ref.transfer.restrict(rk, d), orc.restrict(rk, d))
    fc = ref.transfer.restrict("full", d)
    assert np.array_equal(ref.transfer.prolong(fc), orc.prolong(fc))


@pytest.mark.parametrize("stretch,c,n,sm", [("wall", 3.0, 128, "tweed"),
                                            ("centre", 1.5, 64, "wireframe"),
                                            ("uniform", None, 32, "zebra_alt")])
def test_oracle_solve_bit_exact(ref, orc, stretch, c, n, sm):
    x = ref.grid.make_coords(stretch, n, 1.0, c)
    h = ref.grid.build_hierarchy(x, x)
    f = ref.mgcycle.random_rhs(n, n, 1)
    u, rep = ref.mgcycle.solve(h, ref.mgcycle.CycleConfig(smoother=sm), f)
    uo, repo = orc.solve(orc.Hierarchy(x.values, x.values), f, smoother=sm)
    assert rep.cycles == repo.cycles
    assert rep.defect_norms == repo.defect_norms
    assert np.array_equal(u, uo)


def test_oracle_layouts_match_reference(ref, orc):
    for nx in range(4, 25, 2):
        for ny in range(4, 25, 2):
            for kind, fn in (("tweed", ref.layout.tweed_layout),
                             ("wireframe", ref.layout.wireframe_layout)):
                ii, jj, bb, rr = orc.layout_dump(kind, nx, ny)
                lay = fn(nx, ny)
                k = 0
                for b, blk in enumerate(lay.blocks):
                    for (i, j) in blk.members:
                        assert (ii[k], jj[k], bb[k], rr[k]) == (i, j, b, blk.colour == "red")
                        k += 1
                assert k == len(ii)
