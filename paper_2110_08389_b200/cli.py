"""Command-line front end with the reference's subcommands and report
formats (cli.py:1-214 of the reference):

    python -m paper_2110_08389_b200 solve        --nx N --ny N --smoother K ...
    python -m paper_2110_08389_b200 spectral     --nx N --ny N --smoother K --nu V
    python -m paper_2110_08389_b200 defect-field --nx N --ny N --smoother K ...
    python -m paper_2110_08389_b200 grid         --n N [--stretch S --c C]
    python -m paper_2110_08389_b200 layout       --nx N --ny N --scheme tweed|wireframe

Output contract (kept byte-compatible with the reference): CSV traces with
the header ``cycle,relaxations,defect_max,rel_defect``, JSON documents with
sorted keys and two-space indent, every float printed with 17 significant
digits.  Exit status 0 on completion (flagged non-convergence included), 2
on usage errors (argparse), 1 when an output file cannot be written.  The
solve / spectral / defect-field commands run on the GPU (the library); grid
and layout are host-side setup.
"""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from . import grid, layout, mgcycle, smoothers, transfer


def fmt17(v: float) -> str:
    return format(float(v), ".17g")


class Sink:
    """'-' writes to stdout; anything else is a file path (IO error -> exit 1)."""

    def __init__(self, target: str):
        self.target = target

    def put(self, text: str):
        if self.target == "-":
            sys.stdout.write(text)
            return
        try:
            with open(self.target, "w") as fh:
                fh.write(text)
        except OSError as exc:
            print(f"error: {exc}", file=sys.stderr)
            raise SystemExit(1) from exc


def _json(doc) -> str:
    return json.dumps(doc, sort_keys=True, indent=2) + "\n"


def _csv(header: str, rows) -> str:
    return "\n".join([header] + list(rows)) + "\n"


def _grid_pair(parser, a):
    try:
        return (grid.make_coords(a.stretch, a.nx, a.lx, a.c),
                grid.make_coords(a.stretch, a.ny, a.ly, a.c))
    except ValueError as exc:
        parser.error(str(exc))


# ---------------------------------------------------------------------------
# commands

def run_solve(parser, a) -> int:
    h = grid.build_hierarchy(*_grid_pair(parser, a))
    cfg = mgcycle.CycleConfig(smoother=a.smoother, restriction=a.restrict, nu1=a.nu1,
                              nu2=a.nu2, tol=a.tol, max_cycles=a.max_cycles, seed=a.seed)
    _, rep = mgcycle.solve(h, cfg, mgcycle.random_rhs(a.nx, a.ny, a.seed))
    d = rep.defect_norms
    rows = [f"0,0,{fmt17(d[0])},{fmt17(1.0)}"]
    rows += [f"{k},{rep.relaxations[k - 1]},{fmt17(d[k])},{fmt17(d[k] / d[0])}"
             for k in range(1, len(d))]
    Sink(a.trace).put(_csv("cycle,relaxations,defect_max,rel_defect", rows))
    config = {k: getattr(a, k) for k in ("nx", "ny", "stretch", "c", "smoother", "restrict",
                                          "nu1", "nu2", "tol", "max_cycles", "seed")}
    Sink(a.out).put(_json({"config": config, "converged": rep.converged, "cycles": rep.cycles,
                           "final_rel_defect": rep.final_rel_defect,
                           "per_cycle_ratios": rep.per_cycle_ratios}))
    return 0


def run_spectral(parser, a) -> int:
    from . import spectral
    if a.nu < 1:
        parser.error("--nu must be >= 1")
    h = grid.build_hierarchy(*_grid_pair(parser, a))
    if len(h.levels) < 2:
        parser.error("grid too coarse for a two-grid analysis")
    cfg = spectral.TwoGridConfig(h.levels[0], h.levels[1], smoother=a.smoother,
                                 restriction=a.restrict, nu1=a.nu, nu2=0,
                                 max_iters=a.max_iters, seed=a.seed)
    r = spectral.spectral_radius(cfg)
    Sink(a.out).put(_json({"rho": r.rho, "converged": r.converged,
                           "oscillation": r.oscillation, "iters": r.iters}))
    return 0


def run_defect_field(parser, a) -> int:
    from . import stencil
    h = grid.build_hierarchy(*_grid_pair(parser, a))
    cfg = mgcycle.CycleConfig(smoother=a.smoother, restriction=a.restrict, nu1=a.nu1,
                              nu2=a.nu2, seed=a.seed, tol=1e-300,
                              max_cycles=max(a.cycles, 1))
    f = mgcycle.random_rhs(a.nx, a.ny, a.seed)
    u = np.zeros((a.nx + 1, a.ny + 1))
    state = mgcycle._CycleState(h)
    for _ in range(a.cycles):
        mgcycle.v_cycle(h, cfg, u, f, _state=state)
    d = np.abs(stencil.defect(h.finest.stencil, u, f))
    # one CSV row per j, columns over i (the reference's orientation)
    Sink(a.out).put("\n".join(",".join(fmt17(v) for v in d[:, j]) for j in range(a.ny + 1))
                    + "\n")
    return 0


def run_grid(parser, a) -> int:
    try:
        xs = grid.make_coords(a.stretch, a.n, a.length, a.c).values
    except ValueError as exc:
        parser.error(str(exc))
    Sink(a.out).put(_csv("index,coord", (f"{i},{fmt17(v)}" for i, v in enumerate(xs))))
    return 0


def run_layout(parser, a) -> int:
    build = {"tweed": layout.tweed_layout, "wireframe": layout.wireframe_layout}[a.scheme]
    try:
        lay = build(a.nx, a.ny)
    except ValueError as exc:
        parser.error(str(exc))
    rows = (f"{i},{j},{b},{blk.colour},{lay.scheme}"
            for b, blk in enumerate(lay.blocks) for (i, j) in blk.members)
    Sink(a.out).put(_csv("i,j,block_id,colour,scheme", rows))
    return 0


# ---------------------------------------------------------------------------
# parser

def _stretch(p):
    p.add_argument("--stretch", choices=("uniform", "wall", "centre"), default="uniform")
    p.add_argument("--c", type=float, default=None,
                   help="stretching strength (required for wall/centre)")


def _problem(p):
    p.add_argument("--nx", type=int, required=True)
    p.add_argument("--ny", type=int, required=True)
    p.add_argument("--lx", type=float, default=1.0)
    p.add_argument("--ly", type=float, default=1.0)
    _stretch(p)
    p.add_argument("--smoother", choices=smoothers.KINDS, required=True)
    p.add_argument("--restrict", choices=transfer.RESTRICTIONS, default="full")
    p.add_argument("--seed", type=int, default=0)


COMMANDS = {
    "solve": ("run multigrid V-cycles on a random RHS", run_solve, [
        _problem, ("--nu1", int, 2), ("--nu2", int, 2), ("--tol", float, 1e-10),
        ("--max-cycles", int, 50), ("--trace", str, "-"), ("--out", str, "-")]),
    "spectral": ("two-grid spectral radius", run_spectral, [
        _problem, ("--nu", int, None), ("--max-iters", int, 3000), ("--out", str, "-")]),
    "defect-field": ("dump |defect| after K cycles", run_defect_field, [
        _problem, ("--nu1", int, 2), ("--nu2", int, 2), ("--cycles", int, 3),
        ("--out", str, "-")]),
    "grid": ("dump 1D grid coordinates as CSV", run_grid, [
        ("--n", int, None), ("--length", float, 1.0), _stretch, ("--out", str, "-")]),
    "layout": ("dump block membership as CSV", run_layout, [
        ("--nx", int, None), ("--ny", int, None), ("--scheme", ("tweed", "wireframe"), None),
        ("--out", str, "-")]),
}


def build_parser() -> argparse.ArgumentParser:
    top = argparse.ArgumentParser(prog="tweedmg")
    sub = top.add_subparsers(dest="command", required=True)
    for name, (help_, fn, flags) in COMMANDS.items():
        p = sub.add_parser(name, help=help_)
        for fl in flags:
            if callable(fl):
                fl(p)
                continue
            flag, typ, default = fl
            kw = {"required": True} if default is None else {"default": default}
            if isinstance(typ, tuple):
                p.add_argument(flag, choices=typ, **kw)
            else:
                p.add_argument(flag, type=typ, **kw)
        p.set_defaults(func=fn)
    return top


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    return args.func(parser, args)


if __name__ == "__main__":
    sys.exit(main())
