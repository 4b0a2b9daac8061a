"""Inter-grid transfers on the device (transfer.py of the reference).

Coarse (I, J) sits at fine (2I, 2J).  Full weighting is 1/4 centre, 1/8 edge
neighbours, 1/16 diagonals; half weighting 1/2 and 1/8; prolongation is
bilinear with a zero boundary ring (R_full = P^T / 4).  Both kernels evaluate
in the reference's numpy order and are bit-identical to it.  The V-cycle uses
the fused residual+restriction and prolongation+correction kernels instead
(see mgcycle.py).
"""

from __future__ import annotations

from . import _device, _lib

RESTRICTIONS = ("half", "full")


def _coarse_shape(shape):
    nxp, nyp = shape
    if (nxp - 1) % 2 or (nyp - 1) % 2:
        raise ValueError(f"fine grid {tuple(shape)} cannot be halved")
    return ((nxp - 1) // 2 + 1, (nyp - 1) // 2 + 1)


def restrict(kind: str, d):
    """Restrict a fine defect to the next coarser grid (transfer.py:21-39)."""
    if kind not in RESTRICTIONS:
        raise ValueError(f"unknown restriction kind {kind!r}")
    cshape = _coarse_shape(_device.shape_of(d))
    dd = _device.to_device(d)
    out = _device.empty(cshape)
    nxf, nyf = dd.shape[0] - 1, dd.shape[1] - 1
    _lib.check(_lib.lib().tmg_restrict(nxf, nyf, 1 if kind == "full" else 0, _device.ptr(dd),
                                       _device.ptr(out), _device.stream_handle()))
    return _device.back(out, d)


def prolong(uc):
    """Bilinear interpolation to the next finer grid (transfer.py:42-56)."""
    ncx, ncy = _device.shape_of(uc)
    if min(ncx, ncy) < 3:
        raise ValueError(f"coarse grid {(ncx, ncy)} has no interior to interpolate")
    ud = _device.to_device(uc)
    out = _device.empty((2 * ncx - 1, 2 * ncy - 1))
    _lib.check(_lib.lib().tmg_prolong(ncx - 1, ncy - 1, _device.ptr(ud), _device.ptr(out),
                                      _device.stream_handle()))
    return _device.back(out, uc)
