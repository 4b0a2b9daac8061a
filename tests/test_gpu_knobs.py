"""Library knobs that are read once per process, each exercised in its own
subprocess (tests/knob_worker.py): the strip residual-norm kernel forced
down to small grids (TMG_MARCH_MIN=4), its marching-warp variant (TMG_NORM=1)
and the host-driven solve loop (TMG_SOLVE_HOST=1, the fallback when the
driver refuses conditional graph nodes).  Every norm is compared bit for bit
with the CPU oracle."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{}, {"TMG_MARCH_MIN": "4"},
                                 {"TMG_MARCH_MIN": "4", "TMG_NORM": "1"},
                                 {"TMG_SOLVE_HOST": "1"},
                                 {"TMG_SOLVE_HOST": "1", "TMG_MARCH_MIN": "4"}])
def test_norm_and_solve_knobs(cuda, env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "knob_worker.py")],
                       env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("OK"), r.stdout
