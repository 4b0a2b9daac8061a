"""Subprocess worker for tests/test_gpu_knobs.py: runs under environment knobs
that the library reads once per process (TMG_MARCH_MIN, TMG_NORM,
TMG_SOLVE_HOST) and checks

* the loaded session's residual max-norm (tmg_session_norm, hybrid layout,
  the strip / marching kernels when TMG_MARCH_MIN is small) bit for bit
  against the oracle's defect_max (stencil.py:91-96, mgcycle.py:122,130),
  before and after V-cycles, for the tweed, wireframe and zebra_x layouts
  and sizes that are not multiples of the kernels' 64-wide tiles;
* the solve's defect trace (device while-loop or host fallback) bit for bit
  against the session norms of the same cycles.

Prints "OK <cases>" on success; raises otherwise."""

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2110_08389_b200 import _lib, grid, mgcycle  # noqa: E402
from paper_2110_08389_b200.rng import Lcg64  # noqa: E402

CASES = [("tweed", "wall", 3.0, 70, 70), ("tweed", "wall", 2.0, 130, 66),
         ("tweed", "wall", 2.0, 66, 130), ("wireframe", "centre", 1.5, 70, 70),
         ("wireframe", "centre", 1.5, 134, 68), ("zebra_x", "wall", 2.0, 96, 70),
         ("tweed", "wall", 3.0, 256, 256)]


def main():
    L = _lib.lib()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    n_checked = 0
    for kind, stretch, c, n, m in CASES:
        x = grid.make_coords(stretch, n, 1.0, c)
        y = grid.make_coords(stretch, m, 1.0, c)
        h = grid.build_hierarchy(x, y)
        st = (h.finest.stencil.W, h.finest.stencil.E, h.finest.stencil.S, h.finest.stencil.N)
        ost = orc.assemble(x.values, y.values)
        rng = Lcg64(11)
        f = np.zeros((n + 1, m + 1))
        f[1:-1, 1:-1] = rng.fill((n - 1, m - 1)) - 0.5
        u = np.zeros_like(f)
        u[1:-1, 1:-1] = rng.fill((n - 1, m - 1)) - 0.5
        ud, fd = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
        hn = h.native()
        k = _lib.KIND_IDS[kind]
        _lib.check(L.tmg_session_load(hn, k, P(ud), P(fd), s))
        trace = []
        for cyc in range(4):
            v = ctypes.c_double()
            _lib.check(L.tmg_session_norm(hn, ctypes.byref(v), s))
            cur = torch.empty_like(ud)
            _lib.check(L.tmg_session_store(hn, P(cur), s))
            want = orc.defect_max(ost, cur.cpu().numpy(), f)
            assert v.value == want, (kind, n, m, cyc, v.value, want)
            trace.append(v.value)
            n_checked += 1
            _lib.check(L.tmg_session_cycles(hn, k, 1, 2, 2, 1, s))
        del st
        # the solve from u = 0: its trace equals session norms of the same cycles
        cfg = mgcycle.CycleConfig(smoother=kind, nu1=2, nu2=2, tol=1e-300, max_cycles=3)
        _, rep = mgcycle.solve(h, cfg, fd)
        z = torch.zeros_like(fd)
        _lib.check(L.tmg_session_load(hn, k, P(z), P(fd), s))
        for cyc in range(4):
            v = ctypes.c_double()
            _lib.check(L.tmg_session_norm(hn, ctypes.byref(v), s))
            assert v.value == rep.defect_norms[cyc], (kind, n, m, cyc, v.value,
                                                      rep.defect_norms[cyc])
            _lib.check(L.tmg_session_cycles(hn, k, 1, 2, 2, 1, s))
            n_checked += 1
    print(f"OK {n_checked}")


if __name__ == "__main__":
    main()
