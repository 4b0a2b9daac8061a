"""Exact block Gauss-Seidel sweeps on the device (smoothers.py of the reference).

One sweep unit is a red colour stage then a black one; the alternating kinds
count the pair as one unit (smoothers.py:18-22, 126-133).  Each colour stage
is one launch per block-size class of the block-solver kernel
(csrc/tmg_sweep.cu); block membership comes from the closed-form geometry of
csrc/tmg_plan.cu, compiled once per level and kept on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _device, _lib
from .stencil import native_level

KINDS = ("checkerboard", "zebra_x", "zebra_y", "zebra_alt",
         "tweed", "wireframe", "tweed_wire_alt")
PAIR_KINDS = ("zebra_alt", "tweed_wire_alt")
_BASE = ("checkerboard", "zebra_x", "zebra_y", "tweed", "wireframe")


@dataclass(frozen=True)
class DevicePlan:
    """Handle of the device-resident colour plan of one scheme on one grid.

    The reference's ColourPlan holds flat int64 index arrays per colour
    (smoothers.py:25-34); here the plan is a per-block geometry table built
    natively on first use by the level that sweeps with it."""

    scheme: str
    nx: int
    ny: int


def compile_plan(scheme: str, nx: int, ny: int) -> DevicePlan:
    """Validate and describe the plan of one non-alternating scheme
    (smoothers.py:92-104)."""
    if scheme not in _BASE:
        raise ValueError(f"unknown smoother scheme {scheme!r}")
    if scheme in ("tweed", "wireframe") and (nx < 4 or ny < 4 or nx % 2 or ny % 2):
        raise ValueError(f"block layouts need even nx, ny >= 4, got ({nx}, {ny})")
    return DevicePlan(scheme, nx, ny)


class PlanBundle:
    """Lazy cache of plans for one grid size (smoothers.py:107-118)."""

    def __init__(self, nx: int, ny: int):
        self.nx = nx
        self.ny = ny
        self._plans: dict[str, DevicePlan] = {}

    def plans(self, scheme: str) -> DevicePlan:
        if scheme not in self._plans:
            self._plans[scheme] = compile_plan(scheme, self.nx, self.ny)
        return self._plans[scheme]


def _validate(kind, st, u, f):
    if kind not in KINDS:
        raise ValueError(f"unknown smoother kind {kind!r}")
    want = (st.nx + 1, st.ny + 1)
    if _device.shape_of(u) != want or _device.shape_of(f) != want:
        raise ValueError("field shapes do not match the stencil grid")


def _run(kind, st, bundle, u, f, colour, check):
    _validate(kind, st, u, f)
    if bundle is not None:
        for k in ((kind,) if kind not in PAIR_KINDS else
                  {"zebra_alt": ("zebra_x", "zebra_y"),
                   "tweed_wire_alt": ("tweed", "wireframe")}[kind]):
            bundle.plans(k)
    ud = _device.to_device(u)
    fd = _device.to_device(f)
    L = _lib.lib()
    lv = native_level(st)
    s = _device.stream_handle()
    if colour is None:
        _lib.check(L.tmg_sweep(lv, _lib.KIND_IDS[kind], _device.ptr(ud), _device.ptr(fd), s))
    else:
        _lib.check(L.tmg_sweep_colour(lv, _lib.KIND_IDS[kind], 1 if colour == "red" else 0,
                                      _device.ptr(ud), _device.ptr(fd), s))
    if check:
        _lib.check(L.tmg_level_check(lv, s))
    if _device.is_host(u):
        u[...] = ud.cpu().numpy()


def sweep(kind: str, st, bundle: PlanBundle, u, f, check: bool = True):
    """One sweep unit of `kind`, updating u in place (smoothers.py:121-150).

    After each colour stage the defect vanishes at every point of that colour.
    With check=True (default) the device pivot flags are read back (one stream
    sync) and a vanishing pivot raises SingularSystemError as the reference
    does; check=False keeps the call fully asynchronous."""
    _run(kind, st, bundle, u, f, None, check)


def sweep_colour(kind: str, st, u, f, colour: str, check: bool = True):
    """One colour stage ('red' or 'black') of a non-alternating kind."""
    if kind in PAIR_KINDS:
        raise ValueError("colour stages are defined for non-alternating kinds")
    _run(kind, st, None, u, f, colour, check)


def sweep_cost(kind: str, n: int) -> int:
    """Flops of one sweep unit on an n x n interior, n odd (smoothers.py:153-172;
    PAPER.md:232-238, 302-318)."""
    if n < 3 or n % 2 == 0:
        raise ValueError(f"interior side must be odd and >= 3, got {n}")
    closed = {
        "tweed": 12 * n * n - 10 * n + 11,
        "wireframe": 18 * n * n - 8 * n - 1,
        "checkerboard": 9 * n * n,
        "zebra_x": 12 * n * n,
        "zebra_y": 12 * n * n,
        "zebra_alt": 24 * n * n,
        "tweed_wire_alt": 30 * n * n,
    }
    if kind not in closed:
        raise ValueError(f"unknown smoother kind {kind!r}")
    return closed[kind]
