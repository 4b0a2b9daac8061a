"""BASELINE workloads for the CPU reference arm -- test infrastructure only.

numpy restatement of the seeded synthetic inputs of BASELINE.json's five
configs, so that `bench.py --impl reference` builds its coordinates and
right-hand sides without importing the product package (whose import would
map libtmg_b200.so into the CPU arm).  `tests/test_oracle.py` pins every
array here bit for bit against paper_2110_08389_b200.configs / cube.

Follows:
    lcg_uniform      rng.py:20-40 (Lcg64: state = a*state + c mod 2^64, seeded
                     seed ^ c plus one step, top 53 bits / 2^53)
    coords_*         grid.py:37-102 (tanh wall) and BASELINE config 2/5's sinh
                     centre map
    gaussians_rhs    BASELINE config 3 (the recipe frozen in configs.py)
"""

from __future__ import annotations

import numpy as np

from .oracle import coords_tanh_wall

MULT = 6364136223846793005
INC = 1442695040888963407
_MASK = (1 << 64) - 1


class Lcg:
    def __init__(self, seed):
        self.state = (int(seed) ^ INC) & _MASK
        self.state = (MULT * self.state + INC) & _MASK

    def uniform(self):
        self.state = (MULT * self.state + INC) & _MASK
        return (self.state >> 11) / float(1 << 53)

    def fill(self, n):
        """n uniforms, C order (jump-ahead in blocks of 1024 states)."""
        blk = 1024
        out = np.empty(n, dtype=np.uint64)
        for k in range(min(n, blk)):
            self.state = (MULT * self.state + INC) & _MASK
            out[k] = self.state
        if n > blk:
            a, c = 1, 0
            for _ in range(blk):
                a, c = (MULT * a) & _MASK, (MULT * c + INC) & _MASK
            a, c = np.uint64(a), np.uint64(c)
            with np.errstate(over="ignore"):
                for lo in range(blk, n, blk):
                    hi = min(lo + blk, n)
                    out[lo:hi] = out[lo - blk:hi - blk] * a + c
            self.state = int(out[-1])
        return (out >> np.uint64(11)).astype(np.float64) * (1.0 / float(1 << 53))


def coords_sinh_centre(n, L=1.0, gamma=3.0):
    i = np.arange(n + 1)
    v = (L / 2.0) * (1.0 + np.sinh(gamma * (2.0 * i / n - 1.0)) / np.sinh(gamma))
    v[0], v[n] = 0.0, L
    return v


def uniform_pm1_rhs(n, seed, dim=2):
    f = np.zeros((n + 1,) * dim)
    inner = (slice(1, -1),) * dim
    f[inner] = (2.0 * Lcg(seed).fill((n - 1) ** dim) - 1.0).reshape((n - 1,) * dim)
    return f


def gaussians_rhs(x, y, seed=2, count=16, sigma=0.05):
    rng = Lcg(seed)
    f = np.zeros((len(x), len(y)))
    xi, yj = x[1:-1], y[1:-1]
    acc = np.zeros((len(xi), len(yj)))
    for _ in range(count):
        cx, cy, u1, u2 = (rng.uniform() for _ in range(4))
        amp = np.sqrt(-2.0 * np.log(1.0 - u1)) * np.cos(2.0 * np.pi * u2)
        ex = amp * np.exp(-(xi - cx) ** 2 / (2.0 * sigma * sigma))
        ey = np.exp(-(yj - cy) ** 2 / (2.0 * sigma * sigma))
        acc += np.outer(ex, ey)
    f[1:-1, 1:-1] = acc
    return f


# name -> (default n, coordinate maker, smoother, rhs kind, seed)
CONFIGS = {
    "config1": (128, lambda n: coords_tanh_wall(n, 1.0, 3.0), "tweed", "uniform", 0),
    "config2": (1024, lambda n: coords_sinh_centre(n, 1.0, 3.0), "wireframe", "uniform", 1),
    "config3": (8192, lambda n: coords_tanh_wall(n, 1.0, 4.0), "tweed", "gaussians", 2),
    "config4": (256, lambda n: coords_tanh_wall(n, 1.0, 3.0), "tweed", "uniform3", 3),
    "config5": (1024, lambda n: coords_sinh_centre(n, 1.0, 3.0), "wireframe", "uniform3", 4),
}


def workload(name, n=None):
    """(n, coords, smoother, rhs callable) of a BASELINE config."""
    n0, mk, smoother, kind, seed = CONFIGS[name]
    n = n or n0
    x = mk(n)
    if kind == "gaussians":
        rhs = lambda: gaussians_rhs(x, x, seed)  # noqa: E731
    elif kind == "uniform":
        rhs = lambda: uniform_pm1_rhs(n, seed)  # noqa: E731
    else:
        rhs = lambda: uniform_pm1_rhs(n, seed, dim=3)  # noqa: E731
    return n, x, smoother, rhs


def updates_per_cycle(n, nu, dim=2):
    """(nu1 + nu2) x interior points summed over the injection hierarchy."""
    pts, m = 0, n
    while True:
        pts += (m - 1) ** dim
        if m % 2 or m // 2 < 2:
            break
        m //= 2
    return nu * pts
