"""Golden fixtures of the two-grid analyser from the REFERENCE package
(spectral.py), run in the build container where it is importable:

    python tests/golden/make_spectral_golden.py   -> tests/golden/spectral.npz

Cases: the reference test suite's small dense-oracle configurations (n = 8,
tanh wall c = 2), a probe application of M, the pre/post split at n = 16, and
the paper-scale (n = 128) table configurations of its acceptance criterion 5.
For every case the reference's own spectral_radius result is stored.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref", "src"))

import tweedmg  # noqa: E402
from tweedmg import grid, spectral  # noqa: E402
from tweedmg.rng import Lcg64  # noqa: E402

assert tweedmg.HAVE_EXT, "build the reference's Cython kernels first"

SMALL = [("checkerboard", "full", 1, 0), ("zebra_x", "full", 1, 0),
         ("zebra_alt", "full", 1, 0), ("tweed", "full", 1, 0),
         ("tweed", "full", 1, 1), ("wireframe", "half", 1, 0),
         ("tweed_wire_alt", "full", 2, 0), ("zebra_y", "half", 1, 1)]
SPLIT = [(2, 0), (1, 1), (0, 2)]
PAPER = [("uniform", 0.0, "checkerboard", "full", 1), ("uniform", 0.0, "checkerboard", "half", 1),
         ("uniform", 0.0, "tweed", "full", 3), ("wall", 1.5, "tweed", "full", 2),
         ("wall", 1.5, "zebra_alt", "full", 1), ("wall", 3.0, "tweed", "full", 1),
         ("wall", 3.0, "zebra_alt", "full", 2), ("centre", 1.5, "wireframe", "full", 2),
         ("centre", 1.5, "zebra_alt", "full", 1)]


def pair(kind, n, c):
    x = grid.make_coords(kind, n, 1.0, c if kind != "uniform" else None)
    return grid.Level(x, x), grid.Level(grid.coarsen(x), grid.coarsen(x))


def run(cfg):
    r = spectral.spectral_radius(cfg)
    return np.array([r.rho, float(r.converged), float(r.oscillation), float(r.iters)])


def main():
    out = {}
    fine, coarse = pair("wall", 8, 2.0)
    probe = Lcg64(5).fill(49) - 0.5
    for k, (sm, rs, n1, n2) in enumerate(SMALL):
        cfg = spectral.TwoGridConfig(fine, coarse, smoother=sm, restriction=rs, nu1=n1, nu2=n2)
        out[f"small_{k}"] = run(cfg)
        out[f"small_{k}_apply"] = spectral.two_grid_apply(cfg, probe)
    out["probe"] = probe
    fine, coarse = pair("centre", 16, 1.5)
    for k, (n1, n2) in enumerate(SPLIT):
        cfg = spectral.TwoGridConfig(fine, coarse, smoother="wireframe", restriction="full",
                                     nu1=n1, nu2=n2)
        out[f"split_{k}"] = run(cfg)
    for k, (kind, c, sm, rs, nu) in enumerate(PAPER):
        t0 = time.perf_counter()
        fine, coarse = pair(kind, 128, c)
        cfg = spectral.TwoGridConfig(fine, coarse, smoother=sm, restriction=rs, nu1=nu, nu2=0)
        out[f"paper_{k}"] = run(cfg)
        print(kind, c, sm, rs, nu, out[f"paper_{k}"], f"{time.perf_counter() - t0:.1f}s")
    np.savez_compressed(os.path.join(HERE, "spectral.npz"), **out)


if __name__ == "__main__":
    main()
