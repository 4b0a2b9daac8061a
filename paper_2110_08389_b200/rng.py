"""Seeded 64-bit LCG (rng.py:20-40 of the reference), vectorised.

state <- 6364136223846793005 * state + 1442695040888963407 (mod 2^64),
seeded with seed ^ increment and one warm-up step; a uniform double in [0, 1)
is the top 53 bits of the state.  `fill` produces the same stream as the
scalar recurrence (C order) using block jump-ahead in uint64 numpy
arithmetic, so 10^9-value inputs take seconds instead of minutes.
"""

from __future__ import annotations

import numpy as np

MULT = 6364136223846793005
INC = 1442695040888963407
_MASK = (1 << 64) - 1
_BLOCK = 4096


def _affine_power(k: int):
    """(A, C) with state_{n+k} = A * state_n + C (mod 2^64)."""
    a, c = 1, 0
    for _ in range(k):
        a, c = (MULT * a) & _MASK, (MULT * c + INC) & _MASK
    return a, c


_JUMP = _affine_power(_BLOCK)


class Lcg64:
    """Seeded 64-bit LCG producing uniform doubles in [0, 1)."""

    def __init__(self, seed: int):
        self.state = (int(seed) ^ INC) & _MASK
        self._advance()

    def _advance(self) -> int:
        self.state = (MULT * self.state + INC) & _MASK
        return self.state

    def uniform(self) -> float:
        return (self._advance() >> 11) / float(1 << 53)

    def states(self, n: int) -> np.ndarray:
        """The next n states (uint64), advancing the generator."""
        out = np.empty(n, dtype=np.uint64)
        head = min(n, _BLOCK)
        for k in range(head):
            out[k] = self._advance()
        if n > _BLOCK:
            a, c = np.uint64(_JUMP[0]), np.uint64(_JUMP[1])
            with np.errstate(over="ignore"):
                for lo in range(_BLOCK, n, _BLOCK):
                    hi = min(lo + _BLOCK, n)
                    out[lo:hi] = out[lo - _BLOCK:hi - _BLOCK] * a + c
            self.state = int(out[-1])
        return out

    def advance(self, n: int):
        """Skip n states (jump-ahead by squaring the affine map)."""
        a, c = 1, 0
        pa, pc = MULT, INC
        e = int(n)
        while e:
            if e & 1:
                a, c = (pa * a) & _MASK, (pa * c + pc) & _MASK
            pa, pc = (pa * pa) & _MASK, (pa * pc + pc) & _MASK
            e >>= 1
        self.state = (a * self.state + c) & _MASK

    def fill_device(self, shape):
        """`fill` generated on the GPU (same stream, bit for bit): a CUDA
        float64 tensor; for 10^8 - 10^9-value inputs."""
        from . import _device, _lib
        import torch
        _device.require_cuda()
        n = int(np.prod(shape))
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().tmg_lcg_fill(self.state, n, _device.ptr(out),
                                           _device.stream_handle()))
        self.advance(n)
        return out.reshape(tuple(shape))

    def fill(self, shape) -> np.ndarray:
        """Array of uniform [0, 1) samples in C order."""
        n = int(np.prod(shape))
        s = self.states(n)
        vals = (s >> np.uint64(11)).astype(np.float64) * (1.0 / float(1 << 53))
        return vals.reshape(shape)
