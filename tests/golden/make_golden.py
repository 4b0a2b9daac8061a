"""Generate the golden fixtures of tests/golden from the REFERENCE package.

Run in the build container, where the reference is importable (built into
baseline/_ref by __graft_entry__.build()):

    python tests/golden/make_golden.py

Every array here is produced by the reference's own code (tweedmg, Cython
backend) on seeded inputs; the GPU box, which has no reference, checks the
oracle and the CUDA path against these files.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref", "src"))

import tweedmg  # noqa: E402
from tweedmg import grid, layout, mgcycle, smoothers, stencil, transfer  # noqa: E402
from tweedmg.rng import Lcg64  # noqa: E402

assert tweedmg.HAVE_EXT, "build the reference's Cython kernels first"
KINDS = smoothers.KINDS


def small_cases():
    """3 sweeps of every kind on rectangular and square grids."""
    out = {}
    for (nx, ny) in ((12, 10), (10, 14), (16, 16)):
        for stretch, c in (("wall", 3.0), ("centre", 1.5)):
            x = grid.make_coords(stretch, nx, 1.0, c)
            y = grid.make_coords(stretch, ny, 1.0, c)
            st = stencil.assemble(x, y)
            rng = Lcg64(31)
            f = np.zeros((nx + 1, ny + 1))
            f[1:-1, 1:-1] = rng.fill((nx - 1, ny - 1)) - 0.5
            u0 = np.zeros_like(f)
            u0[1:-1, 1:-1] = rng.fill((nx - 1, ny - 1)) - 0.5
            tag = f"{nx}x{ny}_{stretch}"
            out[f"{tag}_x"] = x.values
            out[f"{tag}_y"] = y.values
            out[f"{tag}_W"], out[f"{tag}_E"] = st.W, st.E
            out[f"{tag}_S"], out[f"{tag}_N"] = st.S, st.N
            out[f"{tag}_f"], out[f"{tag}_u0"] = f, u0
            bundle = smoothers.PlanBundle(nx, ny)
            for kind in KINDS:
                u = u0.copy()
                for _ in range(3):
                    smoothers.sweep(kind, st, bundle, u, f)
                out[f"{tag}_{kind}_u3"] = u
            d = stencil.defect(st, u0, f)
            out[f"{tag}_defect"] = d
            out[f"{tag}_restrict_full"] = transfer.restrict("full", d)
            out[f"{tag}_restrict_half"] = transfer.restrict("half", d)
            out[f"{tag}_prolong"] = transfer.prolong(out[f"{tag}_restrict_full"])
    return out


def layouts():
    out = {}
    for (nx, ny) in ((8, 8), (12, 10), (10, 16), (22, 22)):
        for name, fn in (("tweed", layout.tweed_layout), ("wireframe", layout.wireframe_layout)):
            rows = []
            for b, blk in enumerate(fn(nx, ny).blocks):
                for (i, j) in blk.members:
                    rows.append((i, j, b, 1 if blk.colour == "red" else 0))
            out[f"{name}_{nx}x{ny}"] = np.array(rows, dtype=np.int64)
    return out


def traced_solve(x, f, smoother, nu, tol, max_cycles, trace_cycles=1):
    """mgcycle.solve with the finest iterate recorded after every sweep of
    the first `trace_cycles` cycles (mgcycle.py:89-139, same call sequence)."""
    h = grid.build_hierarchy(x, x)
    state = mgcycle._CycleState(h)
    st = h.finest.stencil
    u = np.zeros_like(f)
    trace = []

    def vcyc(lvl, u, f, record):
        levels = h.levels
        lev = levels[lvl]
        if lvl == len(levels) - 1:
            u[:] = state.coarse.solve(f, g=u)
            return
        for _ in range(nu):
            smoothers.sweep(smoother, lev.stencil, state.bundles[lvl], u, f)
            if record and lvl == 0:
                trace.append(u.copy())
        d = stencil.defect(lev.stencil, u, f)
        fc = transfer.restrict("full", d)
        uc = np.zeros_like(fc)
        vcyc(lvl + 1, uc, fc, record)
        u += transfer.prolong(uc)
        for _ in range(nu):
            smoothers.sweep(smoother, lev.stencil, state.bundles[lvl], u, f)
            if record and lvl == 0:
                trace.append(u.copy())

    d0 = np.abs(stencil.defect(st, u, f)).max()
    norms = [d0]
    cycles = 0
    for cycle in range(1, max_cycles + 1):
        vcyc(0, u, f, cycle <= trace_cycles)
        dn = np.abs(stencil.defect(st, u, f)).max()
        norms.append(dn)
        cycles = cycle
        if dn <= tol * d0:
            break
    return np.array(norms), cycles, trace, u


def config_cases():
    out = {}
    # config 1: 129^2 tanh wall c=3, f = 2*Lcg64(0)-1, tweed V(2,2) to 1e-10
    n = 128
    x = grid.make_tanh_wall(n, 1.0, 3.0)
    f = np.zeros((n + 1, n + 1))
    f[1:-1, 1:-1] = 2.0 * Lcg64(0).fill((n - 1, n - 1)) - 1.0
    norms, cycles, trace, u = traced_solve(x, f, "tweed", 2, 1e-10, 50)
    out["config1_f"] = f
    out["config1_norms"] = norms
    out["config1_cycles"] = np.array(cycles)
    for k, t in enumerate(trace):
        out[f"config1_cycle1_sweep{k}"] = t
    out["config1_u"] = u
    # config 2: 1025^2 sinh centre gamma=3, f = 2*Lcg64(1)-1, wireframe V(2,2)
    n = 1024
    i = np.arange(n + 1)
    v = 0.5 * (1.0 + np.sinh(3.0 * (2.0 * i / n - 1.0)) / np.sinh(3.0))
    v[0], v[n] = 0.0, 1.0
    x = grid.Coords1D(v)
    f = np.zeros((n + 1, n + 1))
    f[1:-1, 1:-1] = 2.0 * Lcg64(1).fill((n - 1, n - 1)) - 1.0
    norms, cycles, _, _ = traced_solve(x, f, "wireframe", 2, 1e-10, 50, trace_cycles=0)
    out["config2_coords"] = v
    out["config2_norms"] = norms
    out["config2_cycles"] = np.array(cycles)
    return out


# rows / columns sampled from the config-2 per-sweep iterates (the full
# 1025^2 fields would be 8 MB each): two residues mod 16 on each axis, so both
# colours of every smoother and both N/T owners of the hybrid layout appear
C2_ROWS = np.array([i for i in range(1, 1024) if i % 16 in (1, 8)])
C2_COLS = np.array([j for j in range(1, 1024) if j % 16 in (3, 10)])


def config2_sweeps():
    """Config 2 (1025^2 wireframe V(2,2)): the finest iterate after each of
    the four finest-level sweeps of cycle 1, sampled on C2_ROWS x C2_COLS,
    plus each full iterate's max |u| (the relative-error scale)."""
    n = 1024
    i = np.arange(n + 1)
    v = 0.5 * (1.0 + np.sinh(3.0 * (2.0 * i / n - 1.0)) / np.sinh(3.0))
    v[0], v[n] = 0.0, 1.0
    x = grid.Coords1D(v)
    f = np.zeros((n + 1, n + 1))
    f[1:-1, 1:-1] = 2.0 * Lcg64(1).fill((n - 1, n - 1)) - 1.0
    _, _, trace, _ = traced_solve(x, f, "wireframe", 2, 1e-300, 1, trace_cycles=1)
    out = {"rows": C2_ROWS, "cols": C2_COLS}
    for k, t in enumerate(trace):
        out[f"sweep{k}"] = t[np.ix_(C2_ROWS, C2_COLS)]
        out[f"sweep{k}_absmax"] = np.array(np.abs(t).max())
    return out


def frozen_grid():
    out = {}
    for kind, c in (("wall", 1.5), ("centre", 1.5), ("wall", 4.0)):
        for n in (4, 16, 64):
            out[f"coords_{kind}_{c}_{n}"] = grid.make_coords(kind, n, 1.0, c).values
    out["lcg_seed12345"] = Lcg64(12345).fill(5000)
    out["random_rhs_8x6_seed3"] = mgcycle.random_rhs(8, 6, seed=3)
    return out


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "config2_sweeps":
        np.savez_compressed(os.path.join(HERE, "config2_sweeps.npz"), **config2_sweeps())
        return
    np.savez_compressed(os.path.join(HERE, "small_sweeps.npz"), **small_cases())
    np.savez_compressed(os.path.join(HERE, "layouts.npz"), **layouts())
    np.savez_compressed(os.path.join(HERE, "grid.npz"), **frozen_grid())
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **config_cases())
    print("golden fixtures written")


if __name__ == "__main__":
    main()
