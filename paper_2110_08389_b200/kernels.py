"""Kernel-backend surface (kernels.py of the reference).

The reference selects between a Cython module and a numpy module
(kernels.py:18-47).  This build has exactly one backend, the sm_100a CUDA
library; there is no CPU fallback, so asking for "python" or "cython" is an
error rather than a silent switch.  The module itself is the active backend
and exposes the reference's per-block entry points (_ckernels.pyx:42-185)
with identical argument order: index arrays, coefficients and fields may be
CUDA tensors or numpy arrays; u is updated in place.
"""

from __future__ import annotations

import sys

import numpy as np

from . import _device, _lib
from .tridiag import SingularSystemError  # noqa: F401

NAME = "cuda"
HAVE_EXT = _lib.available()


def active():
    """The currently selected kernel module (this module)."""
    if not HAVE_EXT:
        raise _lib.NativeLibraryError("the sm_100a library is not built")
    return sys.modules[__name__]


def available() -> list[str]:
    return ["cuda"] if HAVE_EXT else []


def set_backend(name: str) -> str:
    """Select a backend; only 'cuda' exists.  Returns the previous name."""
    if name == "cuda":
        if not HAVE_EXT:
            raise RuntimeError("the CUDA kernels are not available")
        return NAME
    if name in ("python", "cython"):
        raise RuntimeError(f"backend {name!r} is a CPU path and is not part of the B200 build")
    raise ValueError(f"unknown backend {name!r}")


class _HostIdx:
    """Host int64 index array handed to the shims in place (the library
    reads host indices directly: no device copy, no read-back)."""

    def __init__(self, a):
        self.a = np.ascontiguousarray(a, dtype=np.int64)

    def numel(self):
        return self.a.size

    def data_ptr(self):
        return self.a.ctypes.data


def _index(a):
    return _HostIdx(a) if isinstance(a, (np.ndarray, list, tuple)) else \
        _device.to_device(a, dtype=np.int64)


def _common(ii, jj, W, E, S, N, u, f):
    idx = [_index(a) for a in (ii, jj)]
    co = [_device.to_device(a) for a in (W, E, S, N)]
    ud, fd = _device.to_device(u), _device.to_device(f)
    nx, ny = ud.shape[0] - 1, ud.shape[1] - 1
    return idx, co, ud, fd, nx, ny


def _finish(u, ud):
    if _device.is_host(u):
        u[...] = ud.cpu().numpy()


def _call(name, ii, jj, W, E, S, N, u, f):
    (di, dj), co, ud, fd, nx, ny = _common(ii, jj, W, E, S, N, u, f)
    fn = getattr(_lib.lib(), name)
    _lib.check(fn(int(di.numel()), _device.ptr(di), _device.ptr(dj), nx, ny,
                  *[_device.ptr(c) for c in co], _device.ptr(ud), _device.ptr(fd),
                  _device.stream_handle()))
    _finish(u, ud)


def relax_points(ii, jj, W, E, S, N, u, f):
    """Point updates u = (f - sum of neighbours) / C (_ckernels.pyx:42-51)."""
    _call("tmg_relax_points", ii, jj, W, E, S, N, u, f)


def relax_chain(ii, jj, W, E, S, N, u, f):
    """Exact solve of one open chain (_ckernels.pyx:91-103)."""
    _call("tmg_relax_chain", ii, jj, W, E, S, N, u, f)


def relax_ring(ii, jj, W, E, S, N, u, f):
    """Exact solve of one closed ring (_ckernels.pyx:106-141)."""
    _call("tmg_relax_ring", ii, jj, W, E, S, N, u, f)


def relax_legged(ii, jj, offs, bi, bj, W, E, S, N, u, f):
    """Exact solve of one m-legged block around branch (bi, bj)
    (_ckernels.pyx:144-185)."""
    (di, dj), co, ud, fd, nx, ny = _common(ii, jj, W, E, S, N, u, f)
    do = _index(offs)
    _lib.check(_lib.lib().tmg_relax_legged(
        int(di.numel()), _device.ptr(di), _device.ptr(dj), int(do.numel()) - 1, _device.ptr(do),
        int(bi), int(bj), nx, ny, *[_device.ptr(c) for c in co], _device.ptr(ud),
        _device.ptr(fd), _device.stream_handle()))
    _finish(u, ud)
