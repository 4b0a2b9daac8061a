"""Subprocess worker for tests/test_gpu_legk.py (the leg kernel's knobs are
read once per process).  For each square tweed grid: two sweeps on the hybrid
session (the TMA-fed L-shell kernel, csrc/tmg_tweedleg.cu, plus the generic
block kernel for the remaining blocks) against two sweeps through the
natural-layout API path, which the oracle pins (tests/test_gpu_parity.py);
then the same against the CPU oracle itself.  Prints "OK <cases>"."""

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2110_08389_b200 import _lib, grid  # noqa: E402
from paper_2110_08389_b200.rng import Lcg64  # noqa: E402
from paper_2110_08389_b200.stencil import native_level  # noqa: E402


def main(sizes):
    L = _lib.lib()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    done = 0
    for n, stretch, c in sizes:
        x = grid.make_coords(stretch, n, 1.0, c)
        y = grid.make_coords(stretch, n, 1.0, 0.5 * c)  # x and y spacings differ
        h = grid.build_hierarchy(x, y)
        rng = Lcg64(11 + n)
        f = np.zeros((n + 1, n + 1))
        f[1:-1, 1:-1] = rng.fill((n - 1, n - 1)) - 0.5
        u = np.zeros_like(f)
        u[1:-1, 1:-1] = rng.fill((n - 1, n - 1)) - 0.5
        u[0, :], u[-1, :], u[:, 0], u[:, -1] = 0.3, -0.2, 0.1, 0.05
        fd = torch.from_numpy(f).cuda()
        ud = torch.from_numpy(u).cuda()
        ref = ud.clone()
        lv = native_level(h.finest.stencil)
        for _ in range(2):
            _lib.check(L.tmg_sweep(lv, 4, P(ref), P(fd), s))
        hn = h.native()
        _lib.check(L.tmg_session_load(hn, 4, P(ud), P(fd), s))
        _lib.check(L.tmg_session_sweeps(hn, 4, 2, s))
        got = torch.empty_like(ud)
        _lib.check(L.tmg_session_store(hn, P(got), s))
        torch.cuda.synchronize()
        err = float((got - ref).abs().max() / ref.abs().max())
        assert err <= 1e-12, (n, err)
        if n <= 2100:
            st = h.finest.stencil
            uo = u.copy()
            for _ in range(2):
                orc.sweep("tweed", (st.W, st.E, st.S, st.N), uo, f, orc.max_threads())
            g = got.cpu().numpy()
            erro = float(np.abs(g - uo).max() / np.abs(uo).max())
            assert erro <= 1e-12, (n, erro)
            assert np.array_equal(g[0, :], uo[0, :]) and np.array_equal(g[:, -1], uo[:, -1])
        done += 1
    print("OK", done)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "default"
    if which == "small":  # run with TMG_LEGK_NMIN / TMG_LEGK_K0 lowered
        # 38, 72: cross legs whose tip chunk holds a single point (pad 16)
        main([(16, "wall", 2.0), (18, "wall", 2.0), (38, "wall", 2.0), (40, "wall", 3.0),
              (64, "centre", 1.5), (72, "wall", 3.0), (100, "wall", 3.0), (130, "wall", 2.0),
              (256, "wall", 3.0), (600, "wall", 4.0)])
    elif which == "split":  # legs over 128 chunks: blocks split over a cluster
        main([(4400, "wall", 4.0), (4362, "wall", 3.0)])
    else:
        main([(512, "wall", 3.0), (1024, "wall", 4.0), (1026, "centre", 2.0), (2048, "wall", 4.0)])
