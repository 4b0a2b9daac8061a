"""CPU ORACLE driver -- test infrastructure only.

Python/numpy restatement of the reference's host-side driver around the C
restatement in tweed_oracle.c (built to oracle/liboracle.so by
`make -C oracle` / __graft_entry__.build()).  Only tests/, smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module; the
product package never does.

Follows, function by function:
    coords / coarsen / hierarchy   grid.py:37-102, 160-169
    assemble                       stencil.py:48-67
    sweep                          smoothers.py:121-150 (C: orc_sweep)
    defect / defect_max            stencil.py:91-96, mgcycle.py:122,130
    restrict / prolong_add         transfer.py:21-56, mgcycle.py:102
    coarse solve                   stencil.py:129-155 (dense LU in C)
    v_cycle / solve                mgcycle.py:80-139
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

SCHEME_IDS = {"checkerboard": 0, "zebra_x": 1, "zebra_y": 2, "tweed": 4, "wireframe": 5}
KINDS = ("checkerboard", "zebra_x", "zebra_y", "zebra_alt",
         "tweed", "wireframe", "tweed_wire_alt")
PAIRS = {"zebra_alt": ("zebra_x", "zebra_y"), "tweed_wire_alt": ("tweed", "wireframe")}


class OracleSingular(ValueError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"oracle not built: {_LIB_PATH} (run make -C oracle)")
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_long)
        c_long, c_int = ctypes.c_long, ctypes.c_int
        L.orc_sweep.argtypes = [c_int, c_long, c_long, dp, dp, dp, dp, dp, dp, c_int]
        L.orc_defect.argtypes = [c_long, c_long, dp, dp, dp, dp, dp, dp, dp, c_int]
        L.orc_defect_max.argtypes = [c_long, c_long, dp, dp, dp, dp, dp, dp, c_int]
        L.orc_defect_max.restype = ctypes.c_double
        L.orc_restrict.argtypes = [c_int, c_long, c_long, dp, dp]
        L.orc_prolong_add.argtypes = [c_long, c_long, dp, dp]
        L.orc_dense_solve.argtypes = [c_long, c_long, dp, dp, dp, dp, dp, dp]
        L.orc_layout_dump.argtypes = [c_int, c_long, c_long, lp, lp, lp, lp, c_long]
        L.orc_layout_dump.restype = c_long
        for name in ("orc_relax_points", "orc_relax_chain", "orc_relax_ring"):
            getattr(L, name).argtypes = [c_long, lp, lp, dp, dp, dp, dp, dp, dp, c_long]
        L.orc_relax_legged.argtypes = [c_long, lp, lp, c_long, lp, c_long, c_long,
                                       dp, dp, dp, dp, dp, dp, c_long]
        L.orc_max_threads.restype = c_int
        L.orc_group.argtypes = [c_int, c_long, c_long, c_long, c_long]
        L.orc_group.restype = c_long
        L.orc_sweep_part.argtypes = [c_int, c_long, c_long, dp, dp, dp, dp, dp, dp, c_int,
                                     c_long, c_long, c_int]
        _lib = L
    return _lib


def _dp(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _lp(a):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_long))


def _check(status):
    if status == 1:
        raise OracleSingular("zero pivot")
    if status != 0:
        raise ValueError(f"oracle status {status}")


# --------------------------------------------------------------------------
# grid (grid.py:37-102)

def coords_uniform(n, L=1.0):
    return np.arange(n + 1) * (L / n)


def coords_tanh_wall(n, L, c):
    i = np.arange(n + 1)
    v = (L / 2.0) * (1.0 + np.tanh(c * (2.0 * i / n - 1.0)) / np.tanh(c))
    v[0] = 0.0
    v[n] = L
    return v


def coords_tanh_centre(n, L, c):
    i = np.arange(n + 1)
    lo = (L / 2.0) * np.tanh(2.0 * c * i / n) / np.tanh(c)
    hi = (L / 2.0) * (2.0 - np.tanh(c * (2.0 - 2.0 * i / n)) / np.tanh(c))
    v = np.where(i <= n // 2, lo, hi)
    v[0] = 0.0
    v[n] = L
    return v


def coords(kind, n, L=1.0, c=None):
    if kind == "uniform":
        return coords_uniform(n, L)
    if kind == "wall":
        return coords_tanh_wall(n, L, c)
    if kind == "centre":
        return coords_tanh_centre(n, L, c)
    raise ValueError(kind)


def hierarchy_coords(x, y):
    """build_hierarchy (grid.py:160-169): injection coarsening of both axes."""
    levels = [(np.asarray(x, float), np.asarray(y, float))]
    while True:
        lx, ly = levels[-1]
        nx, ny = len(lx) - 1, len(ly) - 1
        if nx % 2 or ny % 2 or nx // 2 < 2 or ny // 2 < 2:
            break
        levels.append((lx[::2].copy(), ly[::2].copy()))
    return levels


def assemble(xv, yv):
    """stencil.py:48-67."""
    nx, ny = len(xv) - 1, len(yv) - 1
    W = np.zeros(nx + 1)
    E = np.zeros(nx + 1)
    hx = np.diff(xv)
    dxc = (xv[2:] - xv[:-2]) / 2.0
    W[1:nx] = 1.0 / (dxc * hx[:-1])
    E[1:nx] = 1.0 / (dxc * hx[1:])
    S = np.zeros(ny + 1)
    N = np.zeros(ny + 1)
    hy = np.diff(yv)
    dyc = (yv[2:] - yv[:-2]) / 2.0
    S[1:ny] = 1.0 / (dyc * hy[:-1])
    N[1:ny] = 1.0 / (dyc * hy[1:])
    return W, E, S, N


# --------------------------------------------------------------------------
# kernels

def sweep(kind, st, u, f, nthreads=1):
    """smoothers.py:121-150, in place on numpy u."""
    if kind in PAIRS:
        for k in PAIRS[kind]:
            sweep(k, st, u, f, nthreads)
        return
    W, E, S, N = st
    nx, ny = len(W) - 1, len(S) - 1
    if u.shape != (nx + 1, ny + 1) or f.shape != u.shape:
        raise ValueError("field shapes do not match the stencil grid")
    _check(lib().orc_sweep(SCHEME_IDS[kind], nx, ny, _dp(W), _dp(E), _dp(S), _dp(N),
                           _dp(u), _dp(f), int(nthreads)))


def sweep_part(kind, st, u, f, red, g0, g1, nthreads=1):
    """One colour stage over the blocks of sharding groups [g0, g1) -- one
    rank's share of smoothers.py:139-150 in a sharded V-cycle."""
    W, E, S, N = st
    nx, ny = len(W) - 1, len(S) - 1
    _check(lib().orc_sweep_part(SCHEME_IDS[kind], nx, ny, _dp(W), _dp(E), _dp(S), _dp(N),
                                _dp(u), _dp(f), int(red), int(g0), int(g1), int(nthreads)))


def group_map(kind, nx, ny):
    """(nx+1, ny+1) int array of every interior point's sharding group
    (0 on the boundary), from the C restatement orc_group."""
    g = np.zeros((nx + 1, ny + 1), dtype=np.int64)
    L, sid = lib(), SCHEME_IDS[kind]
    for i in range(1, nx):
        for j in range(1, ny):
            g[i, j] = L.orc_group(sid, nx, ny, i, j)
    return g


def defect(st, u, f, nthreads=1):
    W, E, S, N = st
    nx, ny = len(W) - 1, len(S) - 1
    d = np.empty_like(u)
    lib().orc_defect(nx, ny, _dp(W), _dp(E), _dp(S), _dp(N), _dp(u), _dp(f), _dp(d),
                     int(nthreads))
    return d


def defect_max(st, u, f, nthreads=1):
    W, E, S, N = st
    nx, ny = len(W) - 1, len(S) - 1
    return float(lib().orc_defect_max(nx, ny, _dp(W), _dp(E), _dp(S), _dp(N), _dp(u),
                                      _dp(f), int(nthreads)))


def restrict(kind, d):
    nxp, nyp = d.shape
    out = np.empty(((nxp - 1) // 2 + 1, (nyp - 1) // 2 + 1))
    _check(lib().orc_restrict(1 if kind == "full" else 0, nxp - 1, nyp - 1, _dp(d),
                              _dp(out)))
    return out


def prolong_add(uc, u):
    ncx, ncy = uc.shape
    lib().orc_prolong_add(ncx - 1, ncy - 1, _dp(uc), _dp(u))


def prolong(uc):
    ncx, ncy = uc.shape
    v = np.zeros((2 * ncx - 1, 2 * ncy - 1))
    prolong_add(np.ascontiguousarray(uc), v)
    return v


def dense_solve(st, f, g=None):
    W, E, S, N = st
    nx, ny = len(W) - 1, len(S) - 1
    u = np.zeros_like(f)
    if g is not None:
        u[0, :] = g[0, :]
        u[-1, :] = g[-1, :]
        u[:, 0] = g[:, 0]
        u[:, -1] = g[:, -1]
    _check(lib().orc_dense_solve(nx, ny, _dp(W), _dp(E), _dp(S), _dp(N), _dp(u),
                                 _dp(np.ascontiguousarray(f))))
    return u


def layout_dump(kind, nx, ny):
    """Per-point (i, j, block, red) in layout.py member order."""
    n = (nx - 1) * (ny - 1)
    arrs = [np.empty(n, dtype=np.int64) for _ in range(4)]
    got = lib().orc_layout_dump(SCHEME_IDS[kind], nx, ny, *[_lp(a) for a in arrs], n)
    if got < 0:
        raise ValueError("bad layout dims")
    return tuple(a[:got] for a in arrs)


# --------------------------------------------------------------------------
# V-cycle driver (mgcycle.py:19-139)

@dataclass
class Report:
    defect_norms: list = field(default_factory=list)
    relaxations: list = field(default_factory=list)
    converged: bool = False
    cycles: int = 0

    @property
    def final_rel_defect(self):
        return self.defect_norms[-1] / self.defect_norms[0]

    @property
    def per_cycle_ratios(self):
        d = self.defect_norms
        return [d[k + 1] / d[k] for k in range(len(d) - 1)]


class Hierarchy:
    def __init__(self, x, y):
        self.levels = hierarchy_coords(x, y)
        self.stencils = [assemble(lx, ly) for lx, ly in self.levels]


def _v_cycle(h, smoother, restriction, nu1, nu2, lvl, u, f, nthreads, trace=None):
    st = h.stencils[lvl]
    if lvl == len(h.levels) - 1:
        u[:] = dense_solve(st, f, g=u)
        return
    for _ in range(nu1):
        sweep(smoother, st, u, f, nthreads)
        if trace is not None and lvl == 0:
            trace.append(u.copy())
    d = defect(st, u, f, nthreads)
    fc = restrict(restriction, d)
    uc = np.zeros_like(fc)
    _v_cycle(h, smoother, restriction, nu1, nu2, lvl + 1, uc, fc, nthreads)
    prolong_add(uc, u)
    for _ in range(nu2):
        sweep(smoother, st, u, f, nthreads)
        if trace is not None and lvl == 0:
            trace.append(u.copy())


def v_cycle(h, u, f, smoother="tweed", restriction="full", nu1=2, nu2=2, nthreads=1,
            trace=None):
    _v_cycle(h, smoother, restriction, nu1, nu2, 0, u, f, nthreads, trace)
    return u


def solve(h, f, smoother="tweed", restriction="full", nu1=2, nu2=2, tol=1e-10,
          max_cycles=50, g=None, nthreads=1):
    W, E, S, N = h.stencils[0]
    nx, ny = len(W) - 1, len(S) - 1
    u = np.zeros((nx + 1, ny + 1))
    if g is not None:
        u[0, :] = g[0, :]
        u[-1, :] = g[-1, :]
        u[:, 0] = g[:, 0]
        u[:, -1] = g[:, -1]
    rep = Report()
    d0 = defect_max(h.stencils[0], u, f, nthreads)
    rep.defect_norms.append(d0)
    if d0 == 0.0:
        rep.converged = True
        return u, rep
    per = (2 if smoother in PAIRS else 1) * (nu1 + nu2)
    for cycle in range(1, max_cycles + 1):
        _v_cycle(h, smoother, restriction, nu1, nu2, 0, u, f, nthreads)
        dn = defect_max(h.stencils[0], u, f, nthreads)
        rep.defect_norms.append(dn)
        rep.relaxations.append(cycle * per)
        rep.cycles = cycle
        if not np.isfinite(dn):
            break
        if dn <= tol * d0:
            rep.converged = True
            break
    return u, rep


def max_threads():
    return int(lib().orc_max_threads())


# --------------------------------------------------------------------------
# two-grid analyser (spectral.py:60-120), test oracle for the device version

def two_grid_apply(xf, yf, e, smoother="tweed", restriction="full", nu1=1, nu2=0):
    """M e for the fine grid (xf, yf) and its injected coarse grid."""
    st = assemble(xf, yf)
    stc = assemble(xf[::2].copy(), yf[::2].copy())
    nx, ny = len(xf) - 1, len(yf) - 1
    u = np.zeros((nx + 1, ny + 1))
    u[1:-1, 1:-1] = np.asarray(e, dtype=float).reshape(nx - 1, ny - 1)
    f0 = np.zeros_like(u)
    for _ in range(nu1):
        sweep(smoother, st, u, f0)
    d = defect(st, u, f0)
    uc = dense_solve(stc, restrict(restriction, d))
    prolong_add(uc, u)
    for _ in range(nu2):
        sweep(smoother, st, u, f0)
    return u[1:-1, 1:-1].ravel()


def spectral_radius(xf, yf, smoother="tweed", restriction="full", nu1=1, nu2=0,
                    max_iters=3000, rel_tol=1e-4, tail_window=30, seed=1):
    """Power iteration with the reference's stopping rules; returns
    (rho, converged, oscillation, iters)."""
    from paper_2110_08389_b200.rng import Lcg64
    n = (len(xf) - 2) * (len(yf) - 2)
    v = Lcg64(seed).fill(n) - 0.5
    v /= np.linalg.norm(v)
    est = []

    def stable(a):
        return a.max() > 0 and (a.max() - a.min()) <= rel_tol * a.max()

    for it in range(1, max_iters + 1):
        w = two_grid_apply(xf, yf, v, smoother, restriction, nu1, nu2)
        r = float(np.linalg.norm(w))
        est.append(r)
        if r < 1e-300:
            return 0.0, True, False, it
        v = w / r
        if len(est) >= tail_window:
            tail = np.array(est[-tail_window:])
            if stable(tail):
                return float(tail[-1]), True, False, it
            if stable(np.sqrt(tail[1:] * tail[:-1])):
                return float(np.exp(np.mean(np.log(tail)))), True, True, it
    tail = np.array(est[-tail_window:])
    return float(np.exp(np.mean(np.log(tail)))), False, False, max_iters
