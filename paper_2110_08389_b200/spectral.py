"""Two-grid error-propagation operator and its spectral radius
(spectral.py of the reference).

    M = S^nu2 (I - P Lc^-1 R Lf) S^nu1

acting on fine-interior error vectors: S is one sweep unit of the smoother on
the homogeneous problem, R / P the restriction and bilinear prolongation, Lc^-1
the exact coarse interior solve (spectral.py:1-17).  Every application runs
on the device through the C ABI -- sweeps (tmg_sweep), residual (tmg_defect),
restriction (tmg_restrict), the coarse direct solve (tmg_direct_solve: a
banded LU inverse for the 63^2 coarse interior of the paper's n = 128
tables), fused prolongation + correction (tmg_prolong_correct) -- and the
power iteration keeps its vector on the device; only the norm of each
iterate comes back to the host for the reference's stopping rules
(spectral.py:92-120: tail window of Rayleigh-quotient estimates, the
geometric-mean rule for a complex dominant pair).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device, _lib, smoothers, stencil, transfer
from .grid import Level
from .rng import Lcg64

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


@dataclass
class TwoGridConfig:
    fine: Level
    coarse: Level
    smoother: str = "tweed"
    restriction: str = "full"
    nu1: int = 1
    nu2: int = 0
    max_iters: int = 3000
    rel_tol: float = 1e-4
    tail_window: int = 30
    seed: int = 1

    _bundle: smoothers.PlanBundle = field(default=None, repr=False)
    _coarse_solver: stencil.DirectSolver = field(default=None, repr=False)
    _work: object = field(default=None, repr=False)

    def __post_init__(self):  # spectral.py:44-50
        if self.nu1 + self.nu2 < 1:
            raise ValueError("need nu1 + nu2 >= 1")
        if (self.coarse.nx * 2, self.coarse.ny * 2) != (self.fine.nx, self.fine.ny):
            raise ValueError("coarse level must halve the fine level")
        if self.smoother not in smoothers.KINDS:
            raise ValueError(f"unknown smoother {self.smoother!r}")
        if self.restriction not in transfer.RESTRICTIONS:
            raise ValueError(f"unknown restriction {self.restriction!r}")
        self._bundle = smoothers.PlanBundle(self.fine.nx, self.fine.ny)
        self._coarse_solver = stencil.DirectSolver(self.coarse.stencil)


class _Workspace:
    """Device fields reused by every application of M."""

    def __init__(self, cfg: TwoGridConfig):
        _device.require_cuda()
        fx, fy, cx, cy = cfg.fine.nx, cfg.fine.ny, cfg.coarse.nx, cfg.coarse.ny
        z = lambda a, b: torch.zeros((a + 1, b + 1), dtype=torch.float64, device="cuda")  # noqa
        self.u, self.f0, self.d = z(fx, fy), z(fx, fy), z(fx, fy)
        self.fc, self.uc = z(cx, cy), z(cx, cy)
        self.scratch = torch.empty(1024, dtype=torch.float64, device="cuda")
        self.fine = stencil.native_level(cfg.fine.stencil)
        self.coarse = stencil.native_level(cfg.coarse.stencil)
        self.kind = _lib.KIND_IDS[cfg.smoother]
        self.full = 1 if cfg.restriction == "full" else 0


def _ws(cfg: TwoGridConfig) -> _Workspace:
    if cfg._work is None:
        cfg._work = _Workspace(cfg)
    return cfg._work


def _apply_inplace(cfg: TwoGridConfig, w: _Workspace):
    """w.u <- M w.u (zero boundary ring kept)."""
    L, s = _lib.lib(), _device.stream_handle()
    P = _device.ptr
    for _ in range(cfg.nu1):
        _lib.check(L.tmg_sweep(w.fine, w.kind, P(w.u), P(w.f0), s))
    # coarse-grid correction of the smoothed error: u += P Lc^-1 R (f0 - Lf u)
    _lib.check(L.tmg_defect(w.fine, P(w.u), P(w.f0), P(w.d), s))
    _lib.check(L.tmg_restrict(cfg.fine.nx, cfg.fine.ny, w.full, P(w.d), P(w.fc), s))
    _lib.check(L.tmg_direct_solve(w.coarse, P(w.uc), P(w.fc), s))
    _lib.check(L.tmg_prolong_correct(cfg.coarse.nx, cfg.coarse.ny, P(w.uc), P(w.u), s))
    for _ in range(cfg.nu2):
        _lib.check(L.tmg_sweep(w.fine, w.kind, P(w.u), P(w.f0), s))


def _check_flags(w: _Workspace):
    _lib.check(_lib.lib().tmg_level_check(w.fine, _device.stream_handle()))


def two_grid_apply(cfg: TwoGridConfig, e):
    """Apply M to a fine-interior error vector (flattened, i-major), the
    reference's spectral.py:60-78.  numpy in -> numpy out; CUDA tensor in ->
    CUDA tensor out."""
    w = _ws(cfg)
    mi, mj = cfg.fine.nx - 1, cfg.fine.ny - 1
    host = isinstance(e, np.ndarray)
    ed = _device.to_device(np.asarray(e, dtype=np.float64) if host else e)
    if ed.numel() != mi * mj:
        raise ValueError(f"error vector has {ed.numel()} entries, expected {mi * mj}")
    w.u.zero_()
    w.u[1:-1, 1:-1] = ed.reshape(mi, mj)
    _apply_inplace(cfg, w)
    _check_flags(w)
    out = w.u[1:-1, 1:-1].reshape(-1).clone()
    return out.cpu().numpy() if host else out


@dataclass
class PowerIterationResult:
    rho: float
    converged: bool
    oscillation: bool
    iters: int
    estimates: list = field(repr=False, default_factory=list)


def _tail_stable(vals: np.ndarray, rel_tol: float) -> bool:
    hi = vals.max()
    lo = vals.min()
    return hi > 0 and (hi - lo) <= rel_tol * hi


def _norm(w: _Workspace) -> float:
    out = ctypes.c_double()
    _lib.check(_lib.lib().tmg_vec_norm2(_device.ptr(w.u), w.u.numel(), _device.ptr(w.scratch),
                                         ctypes.byref(out), _device.stream_handle()))
    return out.value


def spectral_radius(cfg: TwoGridConfig) -> PowerIterationResult:
    """Power iteration for rho(M) with the reference's stopping and
    oscillation rules (spectral.py:92-120)."""
    w = _ws(cfg)
    mi, mj = cfg.fine.nx - 1, cfg.fine.ny - 1
    v = Lcg64(cfg.seed).fill(mi * mj) - 0.5
    v /= np.linalg.norm(v)
    w.u.zero_()
    w.u[1:-1, 1:-1] = torch.from_numpy(v.reshape(mi, mj)).cuda()
    L, s = _lib.lib(), _device.stream_handle()
    estimates = []
    for it in range(1, cfg.max_iters + 1):
        _apply_inplace(cfg, w)
        rho_k = _norm(w)
        estimates.append(rho_k)
        if rho_k < 1e-300:  # operator annihilated the iterate
            _check_flags(w)
            return PowerIterationResult(0.0, True, False, it, estimates)
        _lib.check(L.tmg_vec_scale(_device.ptr(w.u), w.u.numel(), 1.0 / rho_k, s))
        if len(estimates) >= cfg.tail_window:
            tail = np.array(estimates[-cfg.tail_window:])
            if _tail_stable(tail, cfg.rel_tol):
                _check_flags(w)
                return PowerIterationResult(float(tail[-1]), True, False, it, estimates)
            # complex dominant pair: |estimate| oscillates but the two-step
            # geometric mean settles
            gm = np.sqrt(tail[1:] * tail[:-1])
            if _tail_stable(gm, cfg.rel_tol):
                _check_flags(w)
                rho = float(np.exp(np.mean(np.log(tail))))
                return PowerIterationResult(rho, True, True, it, estimates)
    _check_flags(w)
    tail = np.array(estimates[-cfg.tail_window:])
    rho = float(np.exp(np.mean(np.log(tail))))
    return PowerIterationResult(rho, False, False, cfg.max_iters, estimates)
