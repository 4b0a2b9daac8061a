"""Golden outputs of the REFERENCE command-line tool (tweedmg.cli), run in the
build container where it is importable:

    python tests/golden/make_cli_golden.py   -> tests/golden/cli/*.txt

Each case is an argument list; every file written by the case ('--out',
'--trace') is stored as tests/golden/cli/<case>.<flag>.txt.
"""

import contextlib
import io
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref", "src"))

from tweedmg import cli  # noqa: E402

CASES = {
    "grid_wall": ["grid", "--n", "16", "--stretch", "wall", "--c", "3"],
    "grid_centre": ["grid", "--n", "12", "--stretch", "centre", "--c", "1.5"],
    "grid_uniform": ["grid", "--n", "8", "--length", "2"],
    "layout_tweed": ["layout", "--nx", "8", "--ny", "6", "--scheme", "tweed"],
    "layout_wire": ["layout", "--nx", "10", "--ny", "10", "--scheme", "wireframe"],
    "layout_tweed_sq": ["layout", "--nx", "12", "--ny", "12", "--scheme", "tweed"],
    "solve_tweed": ["solve", "--nx", "32", "--ny", "32", "--stretch", "wall", "--c", "3",
                    "--smoother", "tweed"],
    "solve_wire": ["solve", "--nx", "32", "--ny", "16", "--stretch", "centre", "--c", "1.5",
                   "--smoother", "wireframe", "--restrict", "half", "--nu1", "1", "--nu2", "1"],
    "spectral": ["spectral", "--nx", "16", "--ny", "16", "--stretch", "wall", "--c", "2",
                 "--smoother", "tweed", "--nu", "2"],
    "defect": ["defect-field", "--nx", "16", "--ny", "12", "--stretch", "wall", "--c", "2",
               "--smoother", "zebra_alt", "--cycles", "2"],
}


def run_case(args, tmp):
    outs = {}
    argv = list(args)
    for flag in ("--out", "--trace"):
        if args[0] in ("solve",) or flag == "--out":
            path = os.path.join(tmp, flag.strip("-"))
            argv += [flag, path]
            outs[flag.strip("-")] = path
    with contextlib.redirect_stdout(io.StringIO()):
        rc = cli.main(argv)
    assert rc == 0, (args, rc)
    return {k: open(p).read() for k, p in outs.items()}


def main():
    with tempfile.TemporaryDirectory() as tmp:
        for name, args in CASES.items():
            for k, text in run_case(args, tmp).items():
                with open(os.path.join(HERE, "cli", f"{name}.{k}.txt"), "w") as fh:
                    fh.write(text)


if __name__ == "__main__":
    main()
