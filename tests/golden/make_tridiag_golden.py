"""Golden vectors of the line-solver API from the REFERENCE's tridiag module.

Run in the build container (reference sources under baseline/_ref):

    python tests/golden/make_tridiag_golden.py

Seeded, strictly diagonally dominant systems (the kind the block relaxations
produce, tridiag.py:5-7); inputs and the reference's outputs go to
tests/golden/tridiag.npz.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref", "src"))

from tweedmg import tridiag  # noqa: E402


def system(rng, m):
    a = -rng.uniform(0.1, 3.0, m)
    c = -rng.uniform(0.1, 3.0, m)
    b = -(a + c) + rng.uniform(0.05, 2.0, m)
    r = rng.uniform(-1.0, 1.0, m)
    return a, b, c, r


def main():
    rng = np.random.default_rng(20211008)
    out = {}
    sizes = [1, 2, 3, 7, 64, 513]
    out["thomas_sizes"] = np.array(sizes)
    for m in sizes:
        a, b, c, r = system(rng, m)
        out[f"thomas_{m}_abcr"] = np.stack([a, b, c, r])
        out[f"thomas_{m}_x"] = tridiag.thomas(a, b, c, r)
    sizes = [3, 4, 9, 128, 1000]
    out["ring_sizes"] = np.array(sizes)
    for m in sizes:
        a, b, c, r = system(rng, m)
        out[f"ring_{m}_abcr"] = np.stack([a, b, c, r])
        out[f"ring_{m}_x"] = tridiag.circulant_thomas(a, b, c, r)
    cases = [(1, 1), (3, 5), (4, 4, 4, 4), (1, 17, 2, 40, 9, 33)]
    out["legged_ncases"] = np.array(len(cases))
    for q, lens in enumerate(cases):
        legs = [system(rng, p) for p in lens]
        d = -rng.uniform(0.1, 3.0, len(lens))
        dc = -d.sum() + sum(-leg[2][-1] for leg in legs) * 0 + rng.uniform(0.5, 2.0) + np.abs(d).sum()
        rc = rng.uniform(-1.0, 1.0)
        xs, xb = tridiag.m_legged_thomas(legs, d, dc, rc)
        out[f"legged_{q}_lens"] = np.array(lens)
        out[f"legged_{q}_abcr"] = np.concatenate([np.stack(leg) for leg in legs], axis=1)
        out[f"legged_{q}_d"] = d
        out[f"legged_{q}_centre"] = np.array([dc, rc])
        out[f"legged_{q}_x"] = np.concatenate(xs)
        out[f"legged_{q}_xb"] = np.array(xb)
    np.savez_compressed(os.path.join(HERE, "tridiag.npz"), **out)
    print("wrote tridiag.npz with", len(out), "arrays")


if __name__ == "__main__":
    main()
