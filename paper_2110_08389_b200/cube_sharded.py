"""Sharded 3D wireframe V-cycle: BASELINE config 5 across the GPUs of one
box.

The cube's blocks fall into a chain of sharding groups exactly as the 2D
kinds do (sharded.py): a 3D wireframe block -- a shell's frame, a ring of
one of its faces, a face centre -- lies in the shell s = min(i', j', k'),
a point's stencil neighbours lie in shells s-1 .. s+1 and coarse shell S is
fine shell 2S.  A rank owns a contiguous shell range balanced by point
count (outer shells are large, inner ones small), sweeps only its blocks,
swaps two halo shells with each neighbour after every colour stage, and
the coarse tail is replicated.  The protocol (sharded.ShardedSolver) and
the arithmetic (the sm_100a library's tmg_cube_* entry points) are shared
with the single-GPU cube path, so the sharded result is bit-identical to
it.  (SURVEY.md §8(e) sketched i-slabs with a SPIKE solve for the lines
that cross them; shells need neither.)
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device, _lib, cube, sharded
from .mgcycle import CycleReport

SCHEME_IDS = {"tweed": 0, "wireframe": 1}

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


def _check(st):
    cube._check(st)


def group_sizes(scheme: str, n: int) -> np.ndarray:
    """sizes[g] = interior points of shell group g (index 0 unused)."""
    L = _lib.lib()
    sid = SCHEME_IDS[scheme]
    need = L.tmg_cube_group_sizes(sid, n, None, 0)
    if need < 0:
        raise ValueError(L.tmg_cube_last_error().decode())
    out = np.zeros(need, dtype=np.int64)
    L.tmg_cube_group_sizes(sid, n, ctypes.c_void_p(out.ctypes.data), need)
    return out


def group_offsets(scheme: str, n: int, g0: int, g1: int) -> np.ndarray:
    """C-order element offsets of the interior points of groups [g0, g1)."""
    L = _lib.lib()
    sid = SCHEME_IDS[scheme]
    m = L.tmg_cube_group_offsets(sid, n, g0, g1, None, 0)
    if m < 0:
        raise ValueError(L.tmg_cube_last_error().decode())
    out = np.zeros(max(m, 1), dtype=np.int64)
    L.tmg_cube_group_offsets(sid, n, g0, g1, ctypes.c_void_p(out.ctypes.data), m)
    return out[:m]


class NativeCubeShardOps:
    """One rank's cube session (the native hierarchy's level fields); every
    operator is one C-ABI call on the current torch stream."""

    device = "cuda"

    def __init__(self, h: cube.CubeHierarchy, nu1: int = 2, nu2: int = 2):
        _device.require_cuda()
        if h.scheme != "wireframe":
            raise ValueError("only the 3D wireframe shards (BASELINE config 5); "
                             "the 3D tweed (config 4) runs on one GPU")
        self.h, self.nu1, self.nu2 = h, int(nu1), int(nu2)
        self.L = _lib.lib()
        self.dims = []
        n = h.n
        for _ in range(h.levels):
            self.dims.append((n, n))
            n //= 2

    def _s(self):
        return _device.stream_handle()

    def group_sizes(self, kind, nx, ny):
        return group_sizes(self.h.scheme, nx)

    def offsets(self, level, g0, g1):
        n = self.dims[level][0]
        return torch.from_numpy(group_offsets(self.h.scheme, n, g0, g1)).to("cuda")

    def buffer(self, n):
        return torch.empty(n, dtype=torch.float64, device="cuda")

    def load(self, u, f):
        _check(self.L.tmg_cube_load(self.h._h, _device.ptr(u), _device.ptr(f), self._s()))

    def store(self, u):
        _check(self.L.tmg_cube_store(self.h._h, _device.ptr(u), self._s()))

    def gather(self, level, which, idx, out):
        _check(self.L.tmg_cube_gather(self.h._h, level, which, _device.ptr(idx), idx.numel(),
                                      _device.ptr(out), self._s()))

    def scatter(self, level, which, idx, buf):
        _check(self.L.tmg_cube_scatter(self.h._h, level, which, _device.ptr(idx), idx.numel(),
                                       _device.ptr(buf), self._s()))

    def sweep(self, level, red, g0, g1):
        _check(self.L.tmg_cube_sweep_part(self.h._h, level, int(red), g0, g1, self._s()))

    def restrict(self, level, groups=None):  # whole level (groups: a rank's share)
        _check(self.L.tmg_cube_restrict(self.h._h, level, self._s()))

    def prolong(self, level, groups=None):
        _check(self.L.tmg_cube_prolong(self.h._h, level, self._s()))

    def tail(self, level):
        _check(self.L.tmg_cube_tail(self.h._h, level, self.nu1, self.nu2, self._s()))

    def norm(self, g0, g1):
        out = ctypes.c_double()
        st = self.L.tmg_cube_norm_part(self.h._h, g0, g1, ctypes.byref(out), self._s())
        if st == _lib.TMG_SINGULAR:
            return float("nan"), self.L.tmg_cube_last_error().decode()
        _check(st)
        return out.value, None


class CubeShardedSolver(sharded.ShardedSolver):
    """cube.solve / v_cycle with the fine levels split between ranks by
    shells.  Every rank passes the full f; every rank gets the full u."""

    def __init__(self, h, cfg, comm: sharded.Comm | None = None, ops=None, min_groups: int = 4):
        if cfg.smoother != "wireframe" or cfg.restriction != "full":
            raise ValueError("the sharded cube path is the 3D wireframe with full weighting")
        ops = ops or NativeCubeShardOps(h, cfg.nu1, cfg.nu2)
        super().__init__(h, cfg, comm=comm, ops=ops, min_groups=min_groups)

    def solve(self, f, g=None):
        """V-cycles from u = 0 until max|f - Lu| <= tol * d0, a non-finite
        defect or max_cycles (mgcycle.py:107-139 on the cube)."""
        if g is not None:
            raise ValueError("the cube path has homogeneous Dirichlet boundaries")
        cfg = self.cfg
        n = self.dims[0][0]
        want = (n + 1,) * 3
        if tuple(f.shape) != want:
            raise ValueError(f"field shape {tuple(f.shape)} does not match {want}")
        host = isinstance(f, np.ndarray)
        if self.ops.device == "cuda":
            fd = _device.to_device(f)
            u = torch.zeros(want, dtype=torch.float64, device="cuda")
        else:
            fd = np.ascontiguousarray(f, dtype=np.float64)
            u = np.zeros(want)
        self.load(u, fd)
        rep = CycleReport()
        d0 = self.norm()
        rep.defect_norms.append(d0)
        if d0 == 0.0:
            rep.converged = True
        else:
            for cycle in range(1, cfg.max_cycles + 1):
                self.v_cycle()
                dn = self.norm()
                rep.defect_norms.append(dn)
                rep.relaxations.append(cycle * (cfg.nu1 + cfg.nu2))
                rep.cycles = cycle
                if not np.isfinite(dn):
                    break
                if dn <= cfg.tol * d0:
                    rep.converged = True
                    break
        self.store(u)
        if host and self.ops.device == "cuda":
            u = u.cpu().numpy()
        return u, rep


def solve(h, cfg, f, comm: sharded.Comm | None = None):
    """Sharded counterpart of cube.solve over the initialised process group."""
    return CubeShardedSolver(h, cfg, comm).solve(f)
