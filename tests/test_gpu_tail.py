"""The persistent coarse tail (TMG_TAIL=1: one cooperative launch runs the
V-cycle's levels <= TMG_TAIL_NMAX, op by op with grid barriers) gives results
bit-identical to the default path (one graph node per colour stage /
transfer), for tweed, wireframe, zebra and alternating kinds, both
weightings and several (nu1, nu2).  Each setting runs in its own process
(tests/tail_worker.py): the knobs are read once per process."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env):
    e = dict(os.environ)
    e["TMG_MINI"] = "0"  # the shared-memory tail (tests/test_gpu_minitail.py) would take these levels first
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "tail_worker.py")],
                       env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    return [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]


def test_tail_bit_identical(cuda):
    base = _run({"TMG_TAIL": "0"})
    for env in ({"TMG_TAIL": "1"}, {"TMG_TAIL": "1", "TMG_TAIL_CTAS": "3"},
                {"TMG_TAIL": "1", "TMG_TAIL_NMAX": "64"}):
        got = _run(env)
        assert len(got) == len(base) > 0
        for a, b in zip(base, got):
            assert a["finite"] and b["finite"]
            assert a["hash"] == b["hash"], (env, a, b)
