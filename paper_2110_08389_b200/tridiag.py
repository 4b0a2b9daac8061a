"""Error type of the block solvers.

The reference's host Thomas / circulant / m-legged solvers (tridiag.py:30-125)
are the algorithm specification of the device block solver in
csrc/tmg_sweep.cu; on this side only the error type is public.  A vanishing
pivot (|p| < 1e-300, tridiag.py:17-27) is detected on the device, flagged and
raised here.
"""

PIVOT_MIN = 1e-300


class SingularSystemError(ValueError):
    """Raised when elimination encounters a vanishing pivot (tridiag.py:20-21)."""
