"""Exact block Gauss-Seidel sweeps on the device (smoothers.py of the reference).

One sweep unit is a red colour stage then a black one; the alternating kinds
count the pair as one unit (smoothers.py:18-22, 126-133).  Each colour stage
is one launch per block-size class of the block-solver kernel
(csrc/tmg_sweep.cu; the L-shells of large square tweed levels in the hybrid
layout on csrc/tmg_tweedleg.cu); block membership comes from the closed-form
geometry of csrc/tmg_plan.cu, compiled once per level and kept on the device.
The reference's per-colour index plans (compile_plan / PlanBundle) are built
on request for callers that drive the per-block kernels themselves.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device, _lib, layout
from .stencil import native_level

KINDS = ("checkerboard", "zebra_x", "zebra_y", "zebra_alt",
         "tweed", "wireframe", "tweed_wire_alt")
PAIR_KINDS = ("zebra_alt", "tweed_wire_alt")
_BASE = ("checkerboard", "zebra_x", "zebra_y", "tweed", "wireframe")


@dataclass
class ColourPlan:
    """Flat per-colour execution plan (smoothers.py:25-34): merged point
    blocks, then legged, line and ring blocks in construction order, as int64
    index arrays.  The device sweep does not need it (its blocks come from the
    closed-form geometry of csrc/tmg_plan.cu); it is the reference's plan
    object for callers that drive the per-block kernels themselves
    (kernels.relax_*)."""

    points_i: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    points_j: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    legged: list = field(default_factory=list)   # (ii, jj, offs, bi, bj)
    chains: list = field(default_factory=list)   # (ii, jj)
    rings: list = field(default_factory=list)    # (ii, jj)


_KIND_POINT, _KIND_LINE, _KIND_LEGGED, _KIND_RING = range(4)


def _layout_plans(scheme: str, nx: int, ny: int) -> dict:
    """compile_layout (smoothers.py:42-62) over the native member dump
    (layout.member_arrays: blocks in construction order, members legs
    tip -> branch then the branch, rings in traversal order)."""
    ii, jj, bb, fl = layout.member_arrays(scheme, nx, ny)
    ii = ii.astype(np.int64)
    jj = jj.astype(np.int64)
    plans = {"red": ColourPlan(), "black": ColourPlan()}
    points = {"red": [], "black": []}
    starts = np.flatnonzero(np.r_[True, bb[1:] != bb[:-1]])
    ends = np.r_[starts[1:], len(bb)]
    for lo, hi in zip(starts.tolist(), ends.tolist()):
        colour = "red" if fl[lo] & 1 else "black"
        kind = (int(fl[lo]) >> 4) & 3
        plan = plans[colour]
        if kind == _KIND_POINT:
            points[colour].append((lo, hi))
        elif kind == _KIND_LINE:
            plan.chains.append((ii[lo:hi].copy(), jj[lo:hi].copy()))
        elif kind == _KIND_RING:
            plan.rings.append((ii[lo:hi].copy(), jj[lo:hi].copy()))
        else:  # legged: legs concatenated tip -> branch, the branch last
            leg_id = (fl[lo:hi - 1] >> 1) & 7
            counts = np.bincount(leg_id, minlength=int(leg_id.max()) + 1)
            offs = np.zeros(len(counts) + 1, dtype=np.int64)
            np.cumsum(counts, out=offs[1:])
            plan.legged.append((ii[lo:hi - 1].copy(), jj[lo:hi - 1].copy(), offs,
                                int(ii[hi - 1]), int(jj[hi - 1])))
    for colour in ("red", "black"):
        if points[colour]:
            sel = np.concatenate([np.arange(lo, hi) for lo, hi in points[colour]])
            plans[colour].points_i = np.ascontiguousarray(ii[sel])
            plans[colour].points_j = np.ascontiguousarray(jj[sel])
    return plans


def _checkerboard_plan(nx: int, ny: int) -> dict:
    """Red points (i + j even) and black points, i-major (smoothers.py:65-75)."""
    ii, jj = np.meshgrid(np.arange(1, nx, dtype=np.int64), np.arange(1, ny, dtype=np.int64),
                         indexing="ij")
    ii, jj = ii.ravel(), jj.ravel()
    red = (ii + jj) % 2 == 0
    return {c: ColourPlan(points_i=np.ascontiguousarray(ii[m]), points_j=np.ascontiguousarray(jj[m]))
            for c, m in (("red", red), ("black", ~red))}


def _zebra_plan(nx: int, ny: int, axis: str) -> dict:
    """One chain per grid line; red lines have odd j (x) or odd i (y)
    (smoothers.py:78-89)."""
    plans = {"red": ColourPlan(), "black": ColourPlan()}
    if axis == "x":
        along = np.arange(1, nx, dtype=np.int64)
        for j in range(1, ny):
            plans["red" if j % 2 else "black"].chains.append((along, np.full_like(along, j)))
    else:
        along = np.arange(1, ny, dtype=np.int64)
        for i in range(1, nx):
            plans["red" if i % 2 else "black"].chains.append((np.full_like(along, i), along))
    return plans


def _check_scheme(scheme: str, nx: int, ny: int):
    if scheme not in _BASE:
        raise ValueError(f"unknown smoother scheme {scheme!r}")
    if scheme in ("tweed", "wireframe") and (nx < 4 or ny < 4 or nx % 2 or ny % 2):
        raise ValueError(f"block layouts need even nx, ny >= 4, got ({nx}, {ny})")


def compile_plan(scheme: str, nx: int, ny: int) -> dict:
    """{"red": ColourPlan, "black": ColourPlan} of one non-alternating scheme
    (smoothers.py:92-104)."""
    _check_scheme(scheme, nx, ny)
    if scheme == "checkerboard":
        return _checkerboard_plan(nx, ny)
    if scheme in ("zebra_x", "zebra_y"):
        return _zebra_plan(nx, ny, scheme[-1])
    return _layout_plans(scheme, nx, ny)


class PlanBundle:
    """Lazy cache of compiled plans for one grid size (smoothers.py:107-118).
    sweep() never compiles them: the device sweep works from the native
    closed-form geometry, so only callers that read plans pay for them."""

    def __init__(self, nx: int, ny: int):
        self.nx = nx
        self.ny = ny
        self._plans: dict[str, dict] = {}

    def plans(self, scheme: str) -> dict:
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
    if bundle is not None and (bundle.nx, bundle.ny) != (st.nx, st.ny):
        raise ValueError("plan bundle and stencil grid sizes differ")
    for k in ((kind,) if kind not in PAIR_KINDS else
              {"zebra_alt": ("zebra_x", "zebra_y"),
               "tweed_wire_alt": ("tweed", "wireframe")}[kind]):
        _check_scheme(k, st.nx, st.ny)
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
