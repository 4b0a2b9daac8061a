"""3D tweed and wireframe multigrid on cubes (BASELINE configs 4 and 5).

The reference is 2D only; this module carries its
semantics to a third axis -- the 7-point operator of stencil.py:43-96 with
coefficients B, T along k, full weighting and trilinear prolongation as the
tensor products of transfer.py:21-56, the m-legged Thomas of
tridiag.py:84-125 for blocks of up to 6 legs -- on the survey's cube layout
(a point lies on the line along the axis of its unique smallest mirrored
coordinate, from the wall to the first tie point, the branch).  The API
mirrors mgcycle: a hierarchy, ``sweep``, ``defect``, ``v_cycle`` and
``solve`` returning a CycleReport.  ``scheme="wireframe"`` selects the
survey's 3D wireframe layout instead (shell frames of 12 edges and 8
corners, closed rings on the shell faces solved as in _ckernels.pyx:106-141,
face and cube centres as points).  Fields are (n+1)^3 float64 arrays, C
order with k fastest; CUDA tensors stay on the device, numpy arrays come
back as numpy.  The checkers are oracle/tweed3d_oracle.c and
oracle/wire3d_oracle.c.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _device, _lib
from .mgcycle import CycleConfig, CycleReport
from .rng import Lcg64


def _check(st):
    if st == _lib.TMG_OK:
        return
    msg = _lib.lib().tmg_cube_last_error().decode(errors="replace")
    if st == _lib.TMG_SINGULAR:
        from .tridiag import SingularSystemError
        raise SingularSystemError(msg)
    if st == _lib.TMG_BADARG:
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


SCHEMES = ("tweed", "wireframe")


class CubeHierarchy:
    """Levels n, n/2, ... down to 2 of a cube whose three axes use the 1D
    coordinates x (grid.Coords1D or an array of n+1 increasing values);
    ``scheme`` is the block layout the sweeps relax ("tweed" or
    "wireframe")."""

    def __init__(self, x, scheme: str = "tweed"):
        if scheme not in SCHEMES:
            raise ValueError(f"unknown 3D scheme {scheme!r}; expected one of {SCHEMES}")
        _device.require_cuda()
        self.scheme = scheme
        v = np.ascontiguousarray(getattr(x, "values", x), dtype=np.float64)
        self.n = len(v) - 1
        if self.n < 2 or self.n % 2:
            raise ValueError(f"cube needs an even n >= 2, got {self.n}")
        self.x = v
        h = ctypes.c_void_p()
        _check(_lib.lib().tmg_cube_create_scheme(self.n, v.ctypes.data_as(ctypes.c_void_p),
                                                 SCHEMES.index(scheme), ctypes.byref(h)))
        self._h = h
        weakref.finalize(self, _lib.lib().tmg_cube_destroy, h)

    @property
    def levels(self) -> int:
        return _lib.lib().tmg_cube_levels(self._h)

    def blocks(self, level: int = 0):
        """(red, black) block counts of a level."""
        L = _lib.lib()
        return L.tmg_cube_blocks(self._h, level, 1), L.tmg_cube_blocks(self._h, level, 0)

    def interior_points(self) -> int:
        """Interior points summed over the levels (for updates/s)."""
        tot, n = 0, self.n
        for _ in range(self.levels):
            tot += (n - 1) ** 3
            n //= 2
        return tot


def _fields(h: CubeHierarchy, *arrs):
    want = (h.n + 1,) * 3
    out = []
    for a in arrs:
        if tuple(a.shape) != want:
            raise ValueError(f"field shape {tuple(a.shape)} does not match {want}")
        out.append(_device.to_device(a))
    return out


def sweep(h: CubeHierarchy, u, f):
    """One 3D sweep of the hierarchy's scheme (red blocks, then black) in
    place on u."""
    ud, fd = _fields(h, u, f)
    s = _device.stream_handle()
    _check(_lib.lib().tmg_cube_sweep(h._h, _device.ptr(ud), _device.ptr(fd), s))
    if _device.is_host(u):
        u[...] = ud.cpu().numpy()
    return u


def defect(h: CubeHierarchy, u, f):
    ud, fd = _fields(h, u, f)
    d = _device.zeros(ud.shape)
    _check(_lib.lib().tmg_cube_defect(h._h, _device.ptr(ud), _device.ptr(fd), _device.ptr(d),
                                      _device.stream_handle()))
    return _device.back(d, u)


def _check_cfg(h: CubeHierarchy, cfg: CycleConfig):
    if cfg.smoother != h.scheme or cfg.restriction != "full":
        raise ValueError(f"this hierarchy smooths with {h.scheme!r} and full weighting; got "
                         f"smoother={cfg.smoother!r}, restriction={cfg.restriction!r}")


def v_cycle(h: CubeHierarchy, cfg: CycleConfig, u, f):
    """One V(nu1, nu2) cycle in place on u (mgcycle.py:80-104 in 3D)."""
    _check_cfg(h, cfg)
    ud, fd = _fields(h, u, f)
    L, s = _lib.lib(), _device.stream_handle()
    _check(L.tmg_cube_load(h._h, _device.ptr(ud), _device.ptr(fd), s))
    _check(L.tmg_cube_cycles(h._h, cfg.nu1, cfg.nu2, 1, s))
    _check(L.tmg_cube_store(h._h, _device.ptr(ud), s))
    if _device.is_host(u):
        u[...] = ud.cpu().numpy()
    return u


def solve(h: CubeHierarchy, cfg: CycleConfig, f):
    """V-cycles from u = 0 until max|f - Lu| <= tol * d0, a non-finite
    defect or max_cycles (mgcycle.py:107-139 in 3D)."""
    _check_cfg(h, cfg)
    (fd,) = _fields(h, f)
    u = _device.zeros(fd.shape)
    L, s = _lib.lib(), _device.stream_handle()
    _check(L.tmg_cube_load(h._h, _device.ptr(u), _device.ptr(fd), s))
    out = ctypes.c_double()
    _check(L.tmg_cube_norm(h._h, ctypes.byref(out), s))
    rep = CycleReport()
    d0 = out.value
    rep.defect_norms.append(d0)
    if d0 == 0.0:
        rep.converged = True
    else:
        # the cycle loop runs on the device (one while-node graph launch)
        norms = np.zeros(max(cfg.max_cycles, 0) + 1)
        cycles, conv = ctypes.c_int(), ctypes.c_int()
        _check(L.tmg_cube_solve_loop(
            h._h, cfg.nu1, cfg.nu2, float(d0), float(cfg.tol), int(cfg.max_cycles),
            norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(cycles),
            ctypes.byref(conv), s))
        rep.cycles = cycles.value
        rep.defect_norms.extend(float(v) for v in norms[1:rep.cycles + 1])
        rep.relaxations = [k * (cfg.nu1 + cfg.nu2) for k in range(1, rep.cycles + 1)]
        rep.converged = bool(conv.value)
    _check(L.tmg_cube_store(h._h, _device.ptr(u), s))
    return _device.back(u, f), rep


def config4_rhs(n: int, device: bool = True, seed: int = 3):
    """BASELINE config 4 right-hand side: 2 * Lcg64(3).fill((n-1)^3) - 1 on the
    interior, 0 on the boundary."""
    g = Lcg64(seed)
    if device:
        import torch
        f = torch.zeros((n + 1,) * 3, dtype=torch.float64, device="cuda")
        f[1:-1, 1:-1, 1:-1] = 2.0 * g.fill_device((n - 1,) * 3) - 1.0
        return f
    f = np.zeros((n + 1,) * 3)
    f[1:-1, 1:-1, 1:-1] = 2.0 * g.fill((n - 1,) * 3) - 1.0
    return f


def config5_rhs(n: int, device: bool = True):
    """BASELINE config 5 right-hand side: 2 * Lcg64(4).fill((n-1)^3) - 1 on the
    interior, 0 on the boundary (the device fill is the
    jump-ahead generator checked bit-equal against Lcg64)."""
    return config4_rhs(n, device, seed=4)
