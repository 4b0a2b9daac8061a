"""Command-line tool (cli.py; reference cli.py:1-214) against the reference
tool's own outputs (tests/golden/cli, make_cli_golden.py).  grid and layout
are host-side and must match byte for byte; solve / spectral / defect-field
run on the GPU and must match structurally (same lines, cycles, flags) and
numerically (rounding-level differences of the device block solver)."""

import csv
import io
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_cli_golden import CASES  # noqa: E402

GOLD = os.path.join(HERE, "golden", "cli")


def _gold(name, key):
    with open(os.path.join(GOLD, f"{name}.{key}.txt")) as fh:
        return fh.read()


def _run(tmp_path, name):
    from paper_2110_08389_b200 import cli
    args = list(CASES[name])
    outs = {"out": str(tmp_path / "out")}
    if args[0] == "solve":
        outs["trace"] = str(tmp_path / "trace")
    for k, p in outs.items():
        args += [f"--{k}", p]
    assert cli.main(args) == 0
    return {k: open(p).read() for k, p in outs.items()}


@pytest.mark.parametrize("name", [n for n in CASES if n.startswith(("grid", "layout"))])
def test_host_commands_byte_identical(tmp_path, name):
    assert _run(tmp_path, name)["out"] == _gold(name, "out")


def test_usage_errors_exit_2():
    from paper_2110_08389_b200 import cli
    for argv in (["grid", "--n", "7"], ["grid", "--n", "8", "--stretch", "wall"],
                 ["layout", "--nx", "8", "--ny", "8", "--scheme", "zebra"], ["nosuch"]):
        with pytest.raises(SystemExit) as ei:
            cli.main(argv)
        assert ei.value.code == 2


def test_io_error_exit_1(tmp_path):
    from paper_2110_08389_b200 import cli
    with pytest.raises(SystemExit) as ei:
        cli.main(["grid", "--n", "8", "--out", str(tmp_path / "no" / "such" / "file")])
    assert ei.value.code == 1


def _num_close(a, b, rtol):
    return abs(a - b) <= rtol * max(abs(b), 1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["solve_tweed", "solve_wire"])
def test_solve_matches_reference(cuda, tmp_path, name):
    got = _run(tmp_path, name)
    tr_g = list(csv.reader(io.StringIO(got["trace"])))
    tr_r = list(csv.reader(io.StringIO(_gold(name, "trace"))))
    assert tr_g[0] == tr_r[0] and len(tr_g) == len(tr_r)
    d0 = float(tr_r[1][2])
    for a, b in zip(tr_g[1:], tr_r[1:]):
        assert a[:2] == b[:2]
        assert abs(float(a[2]) - float(b[2])) <= 1e-6 * float(b[2]) + 1e-11 * d0
    jg, jr = json.loads(got["out"]), json.loads(_gold(name, "out"))
    assert jg["config"] == jr["config"]
    assert jg["cycles"] == jr["cycles"] and jg["converged"] == jr["converged"]
    assert got["out"].count("\n") == _gold(name, "out").count("\n")


@pytest.mark.gpu
def test_spectral_matches_reference(cuda, tmp_path):
    jg = json.loads(_run(tmp_path, "spectral")["out"])
    jr = json.loads(_gold("spectral", "out"))
    assert sorted(jg) == sorted(jr)
    assert jg["converged"] == jr["converged"] and jg["oscillation"] == jr["oscillation"]
    assert abs(jg["iters"] - jr["iters"]) <= 2
    assert _num_close(jg["rho"], jr["rho"], 1e-8)


@pytest.mark.gpu
def test_defect_field_matches_reference(cuda, tmp_path):
    got = _run(tmp_path, "defect")["out"]
    ref = _gold("defect", "out")
    a = np.array([[float(v) for v in r.split(",")] for r in got.strip().split("\n")])
    b = np.array([[float(v) for v in r.split(",")] for r in ref.strip().split("\n")])
    assert a.shape == b.shape
    assert np.abs(a - b).max() <= 1e-9 * np.abs(b).max()
