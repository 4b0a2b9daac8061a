"""Shared-memory coarse tail (csrc/tmg_minitail.cu): V-cycles of all seven
smoother kinds on small grids against the CPU oracle, with the tail on
(default), off (TMG_MINI=0: every level on the per-stage kernels), limited to
short chains (TMG_MINI_UNIT=4) and forced to take rings and lines of up to 128
points (TMG_MINI_UNIT=128).  Each setting runs in its own process
(tests/minitail_worker.py): the knobs are read once."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{}, {"TMG_MINI": "0"}, {"TMG_MINI_UNIT": "4"},
                                 {"TMG_MINI_UNIT": "128"},
                                 {"TMG_MINI_NMAX": "16", "TMG_MINI_UNIT": "128"}])
def test_mini_tail_vcycles(cuda, env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "minitail_worker.py")],
                       env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("OK"), r.stdout
