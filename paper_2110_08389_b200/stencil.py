"""Five-point variable-coefficient operator (stencil.py of the reference).

Coefficients (stencil.py:1-15): for interior (i, j)
    W[i] u[i-1,j] + E[i] u[i+1,j] + S[j] u[i,j-1] + N[j] u[i,j+1] + C u[i,j],
C = -(W[i] + E[i] + S[j] + N[j]).  `assemble` runs on the host (setup) and is
bit-identical to the reference; `apply`, `defect` and `DirectSolver.solve`
run on the device through the C ABI.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _device, _lib


@dataclass(frozen=True)
class StencilCoeffs:
    """W, E indexed by i (length nx+1), S, N by j (ny+1); zero at the ends."""

    W: np.ndarray
    E: np.ndarray
    S: np.ndarray
    N: np.ndarray
    _native: list = field(default_factory=list, repr=False, compare=False)

    @property
    def nx(self) -> int:
        return len(self.W) - 1

    @property
    def ny(self) -> int:
        return len(self.S) - 1

    def centre(self, i, j):
        """C(i, j), broadcastable over index arrays."""
        return -(self.W[i] + self.E[i] + self.S[j] + self.N[j])


def _axis_coeffs(v: np.ndarray):
    n = len(v) - 1
    lo = np.zeros(n + 1)
    hi = np.zeros(n + 1)
    h = np.diff(v)
    dc = (v[2:] - v[:-2]) / 2.0
    lo[1:n] = 1.0 / (dc * h[:-1])
    hi[1:n] = 1.0 / (dc * h[1:])
    return lo, hi


def assemble(x, y) -> StencilCoeffs:
    """Coefficient arrays from 1D coordinates (stencil.py:48-67)."""
    W, E = _axis_coeffs(np.asarray(x.values, dtype=np.float64))
    S, N = _axis_coeffs(np.asarray(y.values, dtype=np.float64))
    return StencilCoeffs(W, E, S, N)


def native_level(st: StencilCoeffs) -> ctypes.c_void_p:
    """The device level handle of a stencil (created once, freed with it)."""
    if not st._native:
        L = _lib.lib()
        _device.require_cuda()
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (st.W, st.E, st.S, st.N)]
        out = ctypes.c_void_p()
        _lib.check(L.tmg_level_create(st.nx, st.ny, *[_lib.host_ptr(a) for a in arrs],
                                      ctypes.byref(out)))
        st._native.append(out)
        weakref.finalize(st, L.tmg_level_destroy, out)
    return st._native[0]


def _check_shape(st: StencilCoeffs, u):
    if _device.shape_of(u) != (st.nx + 1, st.ny + 1):
        raise ValueError(f"field shape {tuple(u.shape)} does not match grid "
                         f"({st.nx + 1}, {st.ny + 1})")


def apply(st: StencilCoeffs, u):
    """L u on the interior, zero on the boundary ring (stencil.py:76-88)."""
    _check_shape(st, u)
    ud = _device.to_device(u)
    out = _device.empty(ud.shape)
    _lib.check(_lib.lib().tmg_apply(native_level(st), _device.ptr(ud), _device.ptr(out),
                                    _device.stream_handle()))
    return _device.back(out, u)


def defect(st: StencilCoeffs, u, f):
    """d = f - L u on the interior, zero on the boundary (stencil.py:91-96)."""
    _check_shape(st, f)
    _check_shape(st, u)
    ud, fd = _device.to_device(u), _device.to_device(f)
    out = _device.empty(ud.shape)
    _lib.check(_lib.lib().tmg_defect(native_level(st), _device.ptr(ud), _device.ptr(fd),
                                     _device.ptr(out), _device.stream_handle()))
    return _device.back(out, u)


def defect_norm(st: StencilCoeffs, u, f) -> float:
    """max over the interior of |f - L u| (mgcycle.py:122,130); one sync."""
    ud, fd = _device.to_device(u), _device.to_device(f)
    v = ctypes.c_double()
    _lib.check(_lib.lib().tmg_defect_norm(native_level(st), _device.ptr(ud), _device.ptr(fd),
                                          ctypes.byref(v), _device.stream_handle()))
    return v.value


def assemble_dense(st: StencilCoeffs) -> np.ndarray:
    """Dense interior operator, j-outer / i-inner ordering (stencil.py:99-126).
    Host-side helper for oracles and tests; not used by the solver."""
    nx, ny = st.nx, st.ny
    mi, mj = nx - 1, ny - 1
    A = np.zeros((mi * mj, mi * mj))
    for j in range(1, ny):
        for i in range(1, nx):
            k = (j - 1) * mi + (i - 1)
            A[k, k] = st.centre(i, j)
            if i > 1:
                A[k, k - 1] = st.W[i]
            if i < nx - 1:
                A[k, k + 1] = st.E[i]
            if j > 1:
                A[k, k - mi] = st.S[j]
            if j < ny - 1:
                A[k, k + mi] = st.N[j]
    return A


class DirectSolver:
    """Exact interior solve L u = f with Dirichlet data from g
    (stencil.py:129-155).  Factored once on the host at first use (dense,
    j-outer ordering); every solve runs on the device."""

    def __init__(self, st: StencilCoeffs):
        self.st = st
        native_level(st)

    def solve(self, f, g=None):
        st = self.st
        _check_shape(st, f)
        fd = _device.to_device(f)
        u = _device.zeros(fd.shape)
        if g is not None:
            _check_shape(st, g)
            gd = _device.to_device(g)
            u[0, :] = gd[0, :]
            u[-1, :] = gd[-1, :]
            u[:, 0] = gd[:, 0]
            u[:, -1] = gd[:, -1]
        _lib.check(_lib.lib().tmg_direct_solve(native_level(st), _device.ptr(u), _device.ptr(fd),
                                               _device.stream_handle()))
        return _device.back(u, f)


def direct_solve(st: StencilCoeffs, f, g=None):
    return DirectSolver(st).solve(f, g)
