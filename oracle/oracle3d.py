"""CPU ORACLE of the 3D tweed and wireframe V-cycles (test infrastructure
only): ctypes wrapper of tweed3d_oracle.c / wire3d_oracle.c plus the V-cycle driver of mgcycle.py:89-139
restated for cubes.  The reference is 2D only, so this restatement is the
checker of the device 3D path (parity unpinned by the reference; pinned by
property tests in tests/test_3d.py)."""

from __future__ import annotations

import ctypes

import numpy as np

from .oracle import Report, lib


def _decl():
    L = lib()
    if getattr(L, "_o3", False):
        return L
    dp = ctypes.POINTER(ctypes.c_double)
    lp = ctypes.POINTER(ctypes.c_long)
    cl, ci = ctypes.c_long, ctypes.c_int
    L.orc3_sweep.argtypes = [cl] + [dp] * 8 + [ci]
    L.orc3_defect.argtypes = [cl] + [dp] * 9 + [ci]
    L.orc3_restrict.argtypes = [cl, dp, dp]
    L.orc3_prolong_add.argtypes = [cl, dp, dp]
    L.orc3_coarse_solve.argtypes = [dp] * 8
    L.orc3_layout_dump.argtypes = [cl, lp, lp, lp, lp, lp, cl]
    L.orc3_layout_dump.restype = cl
    L.orcw3_sweep.argtypes = [cl] + [dp] * 8 + [ci]
    L.orcw3_sweep_part.argtypes = [cl] + [dp] * 8 + [ci, cl, cl]
    L.orcw3_layout_dump.argtypes = [cl, lp, lp, lp, lp, lp, cl]
    L.orcw3_layout_dump.restype = cl
    L._o3 = True
    return L


def _dp(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check(st):
    if st == 1:
        raise ValueError("zero pivot")
    if st != 0:
        raise ValueError(f"oracle3d status {st}")


def axis_coeffs(v):
    """(lo, hi) couplings of one axis (stencil.py:48-67 per axis)."""
    n = len(v) - 1
    lo, hi = np.zeros(n + 1), np.zeros(n + 1)
    h = np.diff(v)
    dc = (v[2:] - v[:-2]) / 2.0
    lo[1:n] = 1.0 / (dc * h[:-1])
    hi[1:n] = 1.0 / (dc * h[1:])
    return lo, hi


def assemble3(x, y, z):
    W, E = axis_coeffs(np.asarray(x, float))
    S, N = axis_coeffs(np.asarray(y, float))
    B, T = axis_coeffs(np.asarray(z, float))
    return W, E, S, N, B, T


SCHEMES = ("tweed", "wireframe")


def sweep(st, u, f, nthreads=1, scheme="tweed"):
    n = len(st[0]) - 1
    fn = _decl().orc3_sweep if scheme == "tweed" else _decl().orcw3_sweep
    if scheme not in SCHEMES:
        raise ValueError(scheme)
    _check(fn(n, *[_dp(a) for a in st], _dp(u), _dp(f), int(nthreads)))


def sweep_part(st, u, f, red, g0, g1):
    """One colour stage of the 3D wireframe blocks of sharding groups
    [g0, g1) (group = min(i', j', k'))."""
    n = len(st[0]) - 1
    _check(_decl().orcw3_sweep_part(n, *[_dp(a) for a in st], _dp(u), _dp(f), int(red), int(g0),
                                    int(g1)))


def group_map(n, scheme="wireframe"):
    """Sharding group of every node (0 on the boundary): min(i', j', k') for
    the wireframe, max for the tweed."""
    m = np.minimum(np.arange(n + 1), n - np.arange(n + 1))
    a, b, c = np.meshgrid(m, m, m, indexing="ij")
    g = np.minimum(np.minimum(a, b), c) if scheme == "wireframe" else np.maximum(np.maximum(a, b), c)
    g[0, :, :] = g[-1, :, :] = g[:, 0, :] = g[:, -1, :] = g[:, :, 0] = g[:, :, -1] = 0
    return g


def defect(st, u, f, nthreads=1):
    n = len(st[0]) - 1
    d = np.empty_like(u)
    _decl().orc3_defect(n, *[_dp(a) for a in st], _dp(u), _dp(f), _dp(d), int(nthreads))
    return d


def restrict(d):
    nf = d.shape[0] - 1
    out = np.empty((nf // 2 + 1,) * 3)
    _decl().orc3_restrict(nf, _dp(d), _dp(out))
    return out


def prolong_add(uc, u):
    _decl().orc3_prolong_add(uc.shape[0] - 1, _dp(np.ascontiguousarray(uc)), _dp(u))


def layout_dump(n, scheme="tweed"):
    m = (n - 1) ** 3
    arrs = [np.empty(m, dtype=np.int64) for _ in range(5)]
    fn = _decl().orc3_layout_dump if scheme == "tweed" else _decl().orcw3_layout_dump
    got = fn(n, *[a.ctypes.data_as(ctypes.POINTER(ctypes.c_long))
                                        for a in arrs], m)
    return tuple(a[:got] for a in arrs)


class Hierarchy3:
    def __init__(self, x, scheme="tweed"):
        if scheme not in SCHEMES:
            raise ValueError(scheme)
        self.scheme = scheme
        levels = [np.asarray(x, float)]
        while True:
            n = len(levels[-1]) - 1
            if n % 2 or n // 2 < 2:
                break
            levels.append(levels[-1][::2].copy())
        self.coords = levels
        self.stencils = [assemble3(v, v, v) for v in levels]


def _v_cycle(h, nu1, nu2, lvl, u, f, nthreads):
    st = h.stencils[lvl]
    if lvl == len(h.stencils) - 1:
        _check(_decl().orc3_coarse_solve(*[_dp(a) for a in st], _dp(u), _dp(f)))
        return
    for _ in range(nu1):
        sweep(st, u, f, nthreads, h.scheme)
    fc = restrict(defect(st, u, f, nthreads))
    uc = np.zeros_like(fc)
    _v_cycle(h, nu1, nu2, lvl + 1, uc, fc, nthreads)
    prolong_add(uc, u)
    for _ in range(nu2):
        sweep(st, u, f, nthreads, h.scheme)


def v_cycle(h, u, f, nu1=2, nu2=2, nthreads=1):
    _v_cycle(h, nu1, nu2, 0, u, f, nthreads)
    return u


def solve(h, f, nu1=2, nu2=2, tol=1e-10, max_cycles=50, nthreads=1):
    n = len(h.coords[0]) - 1
    u = np.zeros((n + 1,) * 3)
    rep = Report()
    d0 = float(np.abs(defect(h.stencils[0], u, f, nthreads)).max())
    rep.defect_norms.append(d0)
    if d0 == 0.0:
        rep.converged = True
        return u, rep
    for cyc in range(1, max_cycles + 1):
        v_cycle(h, u, f, nu1, nu2, nthreads)
        dn = float(np.abs(defect(h.stencils[0], u, f, nthreads)).max())
        rep.defect_norms.append(dn)
        rep.relaxations.append(cyc * (nu1 + nu2))
        rep.cycles = cyc
        if not np.isfinite(dn):
            break
        if dn <= tol * d0:
            rep.converged = True
            break
    return u, rep
