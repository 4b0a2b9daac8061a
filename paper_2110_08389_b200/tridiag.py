"""Direct solvers for the line and block relaxation systems (tridiag.py:1-125).

Same three functions, argument conventions and errors as the reference's
host module: the standard Thomas algorithm, the periodic (circulant) Thomas
solver of closed rings and the solver of m tridiagonal legs joined at one
branch unknown.  Array conventions (length m): sub-diagonal a (a[0] unused,
except as the wraparound entry of a ring), diagonal b, super-diagonal c, right-hand
side r.  The systems are solved on the device through the C ABI
(``tmg_thomas`` / ``tmg_circulant_thomas`` / ``tmg_legged_thomas``,
csrc/tmg_runtime.cu) in the reference's operation order, so results are
bit-identical to the reference's numpy code; there is no host fallback.
These are the specification functions of the block solvers in
csrc/tmg_sweep.cu and csrc/tmg_tweedleg.cu, one system per call; the sweeps
do not go through them.  A vanishing pivot (|p| < 1e-300, tridiag.py:17-27)
is flagged on the device and raised here.
"""

import ctypes

import numpy as np

PIVOT_MIN = 1e-300


class SingularSystemError(ValueError):
    """Raised when elimination encounters a vanishing pivot (tridiag.py:20-21)."""


def _vec(v, m, name):
    out = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
    if out.shape[0] != m:
        raise ValueError(f"{name} has length {out.shape[0]}, expected {m}")
    return out


def _call(name, *args):
    from . import _device, _lib

    _lib.check(getattr(_lib.lib(), name)(*args, _device.stream_handle()))


def thomas(a, b, c, r) -> np.ndarray:
    """Solve a[k] x[k-1] + b[k] x[k] + c[k] x[k+1] = r[k] (tridiag.py:30-43)."""
    from . import _lib

    m = len(b)
    if m < 1:
        raise IndexError("thomas: empty system")
    aa, bb, cc, rr = (_vec(v, m, n) for v, n in ((a, "a"), (b, "b"), (c, "c"), (r, "r")))
    x = np.empty(m)
    _call("tmg_thomas", m, *(_lib.host_ptr(v) for v in (aa, bb, cc, rr, x)))
    return x


def circulant_thomas(a, b, c, r) -> np.ndarray:
    """Solve the periodic tridiagonal system of a closed ring (tridiag.py:46-81).

    Wraparound entries: a[0] couples x[0] to x[m-1], c[m-1] couples x[m-1]
    to x[0].
    """
    from . import _lib

    m = len(b)
    if m < 3:
        raise ValueError(f"circulant system needs m >= 3, got {m}")
    aa, bb, cc, rr = (_vec(v, m, n) for v, n in ((a, "a"), (b, "b"), (c, "c"), (r, "r")))
    x = np.empty(m)
    _call("tmg_circulant_thomas", m, *(_lib.host_ptr(v) for v in (aa, bb, cc, rr, x)))
    return x


def m_legged_thomas(legs, d, d_centre, r_centre):
    """Solve m tridiagonal legs joined at one branch unknown (tridiag.py:84-125).

    Each leg is a tuple (a, b, c, r) ordered from its tip towards the branch;
    c[-1] couples the leg's innermost point to the branch unknown, d[k] is the
    branch-row coupling to leg k's innermost point and d_centre the branch
    diagonal.  Returns (list of per-leg solution arrays, branch value).
    """
    from . import _lib

    legs = list(legs)
    if len(legs) < 2:
        raise ValueError(f"need m >= 2 legs, got {len(legs)}")
    sizes = [len(leg[1]) for leg in legs]
    if min(sizes) < 1:
        raise IndexError("m_legged_thomas: empty leg")
    offs = np.zeros(len(legs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum(sizes)
    packed = [np.concatenate([_vec(leg[q], p, "abcr"[q]) for leg, p in zip(legs, sizes)])
              for q in range(4)]
    dd = _vec(d, len(legs), "d")
    x = np.empty(int(offs[-1]))
    xb = ctypes.c_double()
    _call("tmg_legged_thomas", len(legs), _lib.host_ptr(offs),
          *(_lib.host_ptr(v) for v in packed), _lib.host_ptr(dd), float(d_centre),
          float(r_centre), _lib.host_ptr(x), ctypes.cast(ctypes.byref(xb), ctypes.c_void_p))
    return [x[offs[k]:offs[k + 1]].copy() for k in range(len(legs))], float(xb.value)
