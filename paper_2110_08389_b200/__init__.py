"""B200-native multigrid V-cycle hot path of arXiv 2110.08389 (tweed and
wireframe relaxation), a drop-in for the reference `tweedmg` package's
solver / smoother / grid API with every operator running in hand-written
sm_100a CUDA kernels behind a C ABI (include/tweedmg_b200.h)."""

from . import grid, layout, stencil, transfer, tridiag  # noqa: F401
from ._lib import available as _available

HAVE_EXT = _available()

from . import kernels, mgcycle, sharded, smoothers, spectral  # noqa: E402,F401

__all__ = [
    "grid", "layout", "mgcycle", "smoothers", "stencil", "transfer", "tridiag",
    "kernels", "sharded", "spectral", "HAVE_EXT",
]

__version__ = "0.1.0"
