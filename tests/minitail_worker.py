"""Subprocess worker for tests/test_gpu_minitail.py: under the TMG_MINI*
knobs of its environment (read once per process), V-cycles of every smoother
kind on small square and rectangular stretched grids — the levels the
shared-memory coarse tail (csrc/tmg_minitail.cu) takes, including hierarchies
that run in it entirely and nonzero Dirichlet data — against the CPU oracle's
V-cycle (mgcycle.py:89-104): three cycles within 1e-10 relative, both
restrictions.  Prints "OK <cases>"."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2110_08389_b200 import grid, mgcycle, smoothers  # noqa: E402
from paper_2110_08389_b200.rng import Lcg64  # noqa: E402

SIZES = [(16, 16), (32, 32), (64, 64), (24, 40), (48, 20), (128, 32), (8, 8), (4, 4)]


def main():
    n_cases = 0
    for kind in smoothers.KINDS:
        for (nx, ny) in SIZES:
            for restriction in ("full", "half"):
                if restriction == "half" and (nx, ny) not in ((32, 32), (24, 40)):
                    continue
                stretch, c = ("centre", 1.5) if "wire" in kind else ("wall", 3.0)
                x = grid.make_coords(stretch, nx, 1.0, c)
                y = grid.make_coords(stretch, ny, 1.0, c)
                h = grid.build_hierarchy(x, y)
                H = orc.Hierarchy(x.values, y.values)
                rng = Lcg64(5 + nx + ny)
                f = np.zeros((nx + 1, ny + 1))
                f[1:-1, 1:-1] = rng.fill((nx - 1, ny - 1)) - 0.5
                u = rng.fill((nx + 1, ny + 1)) - 0.5  # nonzero guess and Dirichlet ring
                cfg = mgcycle.CycleConfig(smoother=kind, nu1=2, nu2=1, restriction=restriction)
                ud, fd = torch.from_numpy(u.copy()).cuda(), torch.from_numpy(f).cuda()
                uo = u.copy()
                for cyc in range(3):
                    mgcycle.v_cycle(h, cfg, ud, fd)
                    orc.v_cycle(H, uo, f, smoother=kind, restriction=restriction, nu1=2, nu2=1)
                    got = ud.cpu().numpy()
                    err = np.abs(got - uo).max() / max(np.abs(uo).max(), 1e-300)
                    assert err <= 1e-10, (kind, nx, ny, restriction, cyc, err)
                    assert np.array_equal(got[0, :], u[0, :]) and np.array_equal(got[:, -1], u[:, -1])
                n_cases += 1
    print(f"OK {n_cases}")


if __name__ == "__main__":
    main()
