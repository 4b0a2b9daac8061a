"""Black-only prolongation (csrc/tmg_transfer_dev.cuh prolong2_tile skip_red):
on square tweed levels of the hybrid layout the V-cycle corrects only the
black points before post-smoothing, because the first red stage overwrites
every red point without reading it (block Gauss-Seidel, _ckernels.pyx:34-39,
144-185; same-colour blocks never touch).  The iterates must be
bit-identical with the full correction (TMG_PROLONG_BLACK=0), on the block
kernel's levels, the leg kernel's and through the shared-memory tail, for
V(2,2), V(1,1) and V(2,0) (no post-smoothing: the full correction is kept)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "black_worker.py")], env=e,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_black_only_prolongation_is_bit_identical(cuda):
    full = _run({"TMG_PROLONG_BLACK": "0"})
    black = _run({})
    assert full.keys() == black.keys()
    for k in full:
        assert full[k] == black[k], k
