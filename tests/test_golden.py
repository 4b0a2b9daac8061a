"""CPU checks against the golden fixtures produced by the reference
(tests/golden/make_golden.py): the oracle and the host-side setup reproduce
the reference bit for bit.  Runs everywhere (no reference, no GPU needed)."""

import os

import numpy as np
import pytest

from paper_2110_08389_b200 import configs, grid, layout, mgcycle, stencil
from paper_2110_08389_b200.rng import Lcg64

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KINDS = ("checkerboard", "zebra_x", "zebra_y", "zebra_alt", "tweed", "wireframe",
         "tweed_wire_alt")


@pytest.fixture(scope="module")
def small():
    return np.load(os.path.join(GOLD, "small_sweeps.npz"))


@pytest.fixture(scope="module")
def cfgs():
    return np.load(os.path.join(GOLD, "configs.npz"))


TAGS = [f"{nx}x{ny}_{s}" for (nx, ny) in ((12, 10), (10, 14), (16, 16))
        for s in ("wall", "centre")]


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_sweeps_match_golden(orc, small, tag):
    st = tuple(small[f"{tag}_{p}"] for p in "WESN")
    f = small[f"{tag}_f"]
    for kind in KINDS:
        u = small[f"{tag}_u0"].copy()
        for _ in range(3):
            orc.sweep(kind, st, u, f)
        assert np.array_equal(u, small[f"{tag}_{kind}_u3"]), kind


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_residual_transfers_match_golden(orc, small, tag):
    st = tuple(small[f"{tag}_{p}"] for p in "WESN")
    d = orc.defect(st, small[f"{tag}_u0"], small[f"{tag}_f"])
    assert np.array_equal(d, small[f"{tag}_defect"])
    assert np.array_equal(orc.restrict("full", d), small[f"{tag}_restrict_full"])
    assert np.array_equal(orc.restrict("half", d), small[f"{tag}_restrict_half"])
    assert np.array_equal(orc.prolong(small[f"{tag}_restrict_full"]), small[f"{tag}_prolong"])


@pytest.mark.parametrize("tag", TAGS)
def test_host_setup_matches_golden(small, tag):
    nx, ny = (int(v) for v in tag.split("_")[0].split("x"))
    stretch = tag.split("_")[1]
    c = 3.0 if stretch == "wall" else 1.5
    x = grid.make_coords(stretch, nx, 1.0, c)
    y = grid.make_coords(stretch, ny, 1.0, c)
    assert np.array_equal(x.values, small[f"{tag}_x"])
    assert np.array_equal(y.values, small[f"{tag}_y"])
    st = stencil.assemble(x, y)
    for p in "WESN":
        assert np.array_equal(getattr(st, p), small[f"{tag}_{p}"])


def test_layouts_match_golden(orc):
    gold = np.load(os.path.join(GOLD, "layouts.npz"))
    for key in gold.files:
        name, dims = key.split("_")
        nx, ny = (int(v) for v in dims.split("x"))
        want = gold[key]
        ii, jj, bb, fl = layout.member_arrays(name, nx, ny)
        got = np.stack([ii, jj, bb, fl & 1], axis=1).astype(np.int64)
        assert np.array_equal(got, want), key
        oi, oj, ob, orr = orc.layout_dump(name, nx, ny)
        assert np.array_equal(np.stack([oi, oj, ob, orr], axis=1), want), key


def test_grid_and_rng_match_golden():
    gold = np.load(os.path.join(GOLD, "grid.npz"))
    for kind, c in (("wall", 1.5), ("centre", 1.5), ("wall", 4.0)):
        for n in (4, 16, 64):
            got = grid.make_coords(kind, n, 1.0, c).values
            assert np.array_equal(got, gold[f"coords_{kind}_{c}_{n}"])
    assert np.array_equal(Lcg64(12345).fill(5000), gold["lcg_seed12345"])
    assert np.array_equal(mgcycle.random_rhs(8, 6, seed=3), gold["random_rhs_8x6_seed3"])


def test_config_inputs_match_golden(cfgs):
    w1 = configs.workload("config1")
    assert np.array_equal(w1.rhs(), cfgs["config1_f"])
    w2 = configs.workload("config2")
    assert np.array_equal(w2.x.values, cfgs["config2_coords"])


def test_oracle_config1_solve_matches_golden(orc, cfgs):
    """BASELINE config 1 (129^2, tweed V(2,2) to 1e-10): 7 cycles, the same
    defect trace and iterate as the reference."""
    w = configs.workload("config1")
    H = orc.Hierarchy(w.x.values, w.x.values)
    u, rep = orc.solve(H, cfgs["config1_f"], smoother="tweed", tol=1e-10)
    assert rep.cycles == int(cfgs["config1_cycles"]) == 7
    assert np.array_equal(np.array(rep.defect_norms), cfgs["config1_norms"])
    assert np.array_equal(u, cfgs["config1_u"])


def test_oracle_config1_cycle1_sweeps_match_golden(orc, cfgs):
    w = configs.workload("config1")
    H = orc.Hierarchy(w.x.values, w.x.values)
    trace = []
    u = np.zeros_like(cfgs["config1_f"])
    orc.v_cycle(H, u, cfgs["config1_f"], smoother="tweed", trace=trace)
    assert len(trace) == 4
    for k, t in enumerate(trace):
        assert np.array_equal(t, cfgs[f"config1_cycle1_sweep{k}"])


def test_oracle_config2_solve_matches_golden(orc, cfgs):
    """BASELINE config 2 (1025^2 sinh centre, wireframe V(2,2)): 20 cycles."""
    w = configs.workload("config2")
    H = orc.Hierarchy(w.x.values, w.x.values)
    f = w.rhs()
    _, rep = orc.solve(H, f, smoother="wireframe", tol=1e-10, nthreads=orc.max_threads())
    assert rep.cycles == int(cfgs["config2_cycles"]) == 20
    assert np.array_equal(np.array(rep.defect_norms), cfgs["config2_norms"])


def test_oracle_config2_cycle1_sweeps_match_golden(orc):
    """Config 2's four finest-level iterates of cycle 1 (sampled rows/columns
    of the reference's fields, tests/golden/config2_sweeps.npz): the oracle is
    bit-identical to the reference there too."""
    gold = np.load(os.path.join(GOLD, "config2_sweeps.npz"))
    w = configs.workload("config2")
    H = orc.Hierarchy(w.x.values, w.x.values)
    trace = []
    u = np.zeros((1025, 1025))
    orc.v_cycle(H, u, w.rhs(), smoother="wireframe", trace=trace, nthreads=orc.max_threads())
    assert len(trace) == 4
    rows, cols = gold["rows"], gold["cols"]
    for k, t in enumerate(trace):
        assert np.array_equal(t[np.ix_(rows, cols)], gold[f"sweep{k}"])
        assert np.abs(t).max() == gold[f"sweep{k}_absmax"]


def test_oracle_workloads_match_package():
    """oracle/workloads.py (the CPU reference arm's inputs, no product
    import) produces the package's BASELINE inputs bit for bit."""
    from oracle import workloads as wl
    from paper_2110_08389_b200 import cube
    for name, n in (("config1", None), ("config2", 64), ("config3", 256)):
        w = configs.workload(name, n=n)
        nn, x, smoother, rhs = wl.workload(name, n)
        assert nn == w.n and smoother == w.smoother
        assert np.array_equal(x, w.x.values)
        assert np.array_equal(rhs(), w.rhs())
    for name, fn in (("config4", cube.config4_rhs), ("config5", cube.config5_rhs)):
        nn, x, _, rhs = wl.workload(name, 16)
        assert np.array_equal(rhs(), fn(16, device=False))
        want = (configs.sinh_centre(16, 1.0, 3.0) if name == "config5"
                else grid.make_tanh_wall(16, 1.0, 3.0)).values
        assert np.array_equal(x, want)
    assert wl.updates_per_cycle(128, 4) == 4 * sum((m - 1) ** 2 for m in (128, 64, 32, 16, 8, 4, 2))
