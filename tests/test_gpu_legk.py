"""The TMA-fed tweed L-shell kernel (csrc/tmg_tweedleg.cu): sweeps on the
hybrid session agree with the natural-layout block solver and with the CPU
oracle (relax_legged, _ckernels.pyx:144-185) to 1e-12, for the default
configuration, for tiny grids and shells (knobs lowered: one-chunk legs,
many blocks per CTA), and for blocks split over the two CTAs of a cluster."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("which,env", [
    ("default", {}),
    ("small", {"TMG_LEGK_NMIN": "16", "TMG_LEGK_K0": "3"}),
    ("small", {"TMG_LEGK_NMIN": "16", "TMG_LEGK_K0": "9"}),
    ("split", {}),
])
def test_leg_kernel_sweeps(cuda, which, env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "legk_worker.py"), which],
                       env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("OK"), r.stdout
