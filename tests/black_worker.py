"""Subprocess worker for tests/test_gpu_black.py: two tweed V(2,2) cycles (and a
V(1,1) and a V(2,0) cycle) on square grids from a random guess; prints one
SHA-256 of the iterates per case.  The caller runs it with and without
TMG_PROLONG_BLACK (read once per process)."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2110_08389_b200 import grid, mgcycle  # noqa: E402
from paper_2110_08389_b200.rng import Lcg64  # noqa: E402

out = {}
for n, nu1, nu2 in ((64, 2, 2), (256, 2, 2), (256, 1, 1), (256, 2, 0), (1024, 2, 2), (2048, 2, 1)):
    x = grid.make_coords("wall", n, 1.0, 3.0)
    h = grid.build_hierarchy(x, x)
    rng = Lcg64(n)
    f = np.zeros((n + 1, n + 1))
    f[1:-1, 1:-1] = rng.fill((n - 1, n - 1)) - 0.5
    u = rng.fill((n + 1, n + 1)) - 0.5
    ud, fd = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
    cfg = mgcycle.CycleConfig(smoother="tweed", nu1=nu1, nu2=nu2)
    for _ in range(2):
        mgcycle.v_cycle(h, cfg, ud, fd)
    out[f"{n}_{nu1}_{nu2}"] = hashlib.sha256(ud.cpu().numpy().tobytes()).hexdigest()
print(json.dumps(out))
