"""GPU parity against the reference's golden fixtures and, at BASELINE sizes,
against the pinned CPU oracle.  Gates (BASELINE.json north star): per-sweep
iterates within 1e-10 relative, identical V-cycle counts, asymptotic
convergence factors within 1e-3."""

import os

import numpy as np
import pytest

from paper_2110_08389_b200 import configs, grid, mgcycle, smoothers, stencil, transfer
from paper_2110_08389_b200.rng import Lcg64

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KINDS = smoothers.KINDS
TAGS = [f"{nx}x{ny}_{s}" for (nx, ny) in ((12, 10), (10, 14), (16, 16))
        for s in ("wall", "centre")]


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


@pytest.fixture(scope="module")
def cfgs():
    return np.load(os.path.join(GOLD, "configs.npz"))


@pytest.mark.parametrize("tag", TAGS)
def test_sweeps_match_golden(cuda, tag):
    small = np.load(os.path.join(GOLD, "small_sweeps.npz"))
    st = stencil.StencilCoeffs(*(small[f"{tag}_{p}"] for p in "WESN"))
    nx, ny = st.nx, st.ny
    f = cuda.from_numpy(small[f"{tag}_f"]).cuda()
    for kind in KINDS:
        u = cuda.from_numpy(small[f"{tag}_u0"].copy()).cuda()
        for _ in range(3):
            smoothers.sweep(kind, st, smoothers.PlanBundle(nx, ny), u, f)
        assert _rel(u.cpu().numpy(), small[f"{tag}_{kind}_u3"]) <= 1e-12, kind
    d = stencil.defect(st, small[f"{tag}_u0"], small[f"{tag}_f"])
    assert np.array_equal(d, small[f"{tag}_defect"])
    assert np.array_equal(transfer.restrict("full", d), small[f"{tag}_restrict_full"])
    assert np.array_equal(transfer.prolong(small[f"{tag}_restrict_full"]), small[f"{tag}_prolong"])


def test_config1_solve(cuda, cfgs):
    """129^2 tweed V(2,2) to 1e-10: 7 cycles as the reference."""
    w = configs.workload("config1")
    h = grid.build_hierarchy(w.x, w.x)
    cfg = mgcycle.CycleConfig(smoother="tweed", tol=1e-10)
    u, rep = mgcycle.solve(h, cfg, cfgs["config1_f"])
    assert rep.converged and rep.cycles == int(cfgs["config1_cycles"]) == 7
    assert rep.defect_norms[0] == cfgs["config1_norms"][0]
    gold = cfgs["config1_norms"]
    for a, b in zip(rep.defect_norms, gold):
        assert abs(a - b) <= 1e-5 * b + 1e-12 * gold[0]
    assert _rel(u, cfgs["config1_u"]) <= 1e-10


def _cycle1_sweeps(cuda, w, kind, f_host):
    """Cycle 1 of a workload assembled from the public device operators; the
    finest iterate after each of its four sweeps (mgcycle.py:89-104)."""
    h = grid.build_hierarchy(w.x, w.x)
    cfg = mgcycle.CycleConfig(smoother=kind)
    fine = h.finest
    f = cuda.from_numpy(f_host).cuda()
    u = cuda.zeros_like(f)
    bundle = smoothers.PlanBundle(fine.nx, fine.ny)
    got = []
    for _ in range(2):
        smoothers.sweep(kind, fine.stencil, bundle, u, f)
        got.append(u.cpu().numpy())
    fc = transfer.restrict("full", stencil.defect(fine.stencil, u, f))
    uc = cuda.zeros_like(fc)
    mgcycle.v_cycle(grid.Hierarchy(h.levels[1:]), cfg, uc, fc)
    u += transfer.prolong(uc)
    for _ in range(2):
        smoothers.sweep(kind, fine.stencil, bundle, u, f)
        got.append(u.cpu().numpy())
    return got


def test_config1_cycle1_per_sweep(cuda, cfgs):
    """Config 1: the four cycle-1 iterates against the reference's."""
    got = _cycle1_sweeps(cuda, configs.workload("config1"), "tweed", cfgs["config1_f"])
    for k, g in enumerate(got):
        assert _rel(g, cfgs[f"config1_cycle1_sweep{k}"]) <= 1e-10, k


def test_config2_cycle1_per_sweep(cuda):
    """Config 2 (1025^2 wireframe): the four cycle-1 iterates against the
    reference's (sampled rows x columns, tests/golden/config2_sweeps.npz),
    relative to each full iterate's max |u|, gate 1e-10."""
    gold = np.load(os.path.join(GOLD, "config2_sweeps.npz"))
    w = configs.workload("config2")
    got = _cycle1_sweeps(cuda, w, "wireframe", w.rhs())
    rows, cols = gold["rows"], gold["cols"]
    for k, g in enumerate(got):
        scale = float(gold[f"sweep{k}_absmax"])
        assert abs(np.abs(g).max() - scale) <= 1e-10 * scale, k
        err = np.abs(g[np.ix_(rows, cols)] - gold[f"sweep{k}"]).max() / scale
        assert err <= 1e-10, (k, err)


def _asymptotic_ratio(norms, floor=1e-9):
    """test_acceptance.py:316-322 (geometric mean, first two ratios skipped)."""
    d = np.asarray(norms) / norms[0]
    r = [d[k + 1] / d[k] for k in range(len(d) - 1) if d[k + 1] > floor]
    use = r[2:] if len(r) > 3 else r
    return float(np.exp(np.mean(np.log(use))))


def test_config2_solve(cuda, cfgs):
    """1025^2 sinh-centre wireframe V(2,2) to 1e-10: 20 cycles."""
    w = configs.workload("config2")
    h = grid.build_hierarchy(w.x, w.x)
    cfg = mgcycle.CycleConfig(smoother="wireframe", tol=1e-10)
    u, rep = mgcycle.solve(h, cfg, w.rhs())
    assert rep.converged and rep.cycles == int(cfgs["config2_cycles"]) == 20
    gold = cfgs["config2_norms"]
    assert rep.defect_norms[0] == gold[0]
    assert abs(_asymptotic_ratio(rep.defect_norms) - _asymptotic_ratio(gold)) <= 1e-3


@pytest.fixture(scope="module")
def config3(cuda):
    w = configs.workload("config3")
    return w, w.rhs()


def test_config3_sweep_and_cycles_match_oracle(cuda, orc, config3):
    """8193^2, tanh wall gamma=4, 16 Gaussians: one tweed sweep and two
    V(2,2) cycles against the oracle (multi-threaded, bit-identical to the
    reference) at full size."""
    w, f = config3
    nthreads = orc.max_threads()
    h = grid.build_hierarchy(w.x, w.x)
    st = h.finest.stencil
    fd = cuda.from_numpy(f).cuda()
    u = cuda.zeros_like(fd)
    smoothers.sweep("tweed", st, smoothers.PlanBundle(8192, 8192), u, fd)
    uo = np.zeros_like(f)
    orc.sweep("tweed", (st.W, st.E, st.S, st.N), uo, f, nthreads)
    assert _rel(u.cpu().numpy(), uo) <= 1e-10
    del u
    H = orc.Hierarchy(w.x.values, w.x.values)
    ug = cuda.zeros_like(fd)
    uo = np.zeros_like(f)
    cfg = mgcycle.CycleConfig(smoother="tweed", nu1=2, nu2=2)
    for _ in range(2):
        mgcycle.v_cycle(h, cfg, ug, fd)
        orc.v_cycle(H, uo, f, nthreads=nthreads)
        assert _rel(ug.cpu().numpy(), uo) <= 1e-10


def test_wireframe_8193_sweep_and_cycle(cuda, orc):
    """Wireframe at 8193^2 (centre-clustered): the outer rings hold ~2050
    chunks and run on 16-CTA clusters.  One sweep on the API layout and one
    V(2,2) cycle (hybrid layout) against the oracle."""
    n = 8192
    x = grid.make_coords("centre", n, 1.0, 3.0)
    h = grid.build_hierarchy(x, x)
    st = h.finest.stencil
    f = np.zeros((n + 1, n + 1))
    f[1:-1, 1:-1] = Lcg64(4).fill((n - 1, n - 1)) * 2.0 - 1.0
    nthreads = orc.max_threads()
    fd = cuda.from_numpy(f).cuda()
    u = cuda.zeros_like(fd)
    smoothers.sweep("wireframe", st, smoothers.PlanBundle(n, n), u, fd)
    uo = np.zeros_like(f)
    orc.sweep("wireframe", (st.W, st.E, st.S, st.N), uo, f, nthreads)
    assert _rel(u.cpu().numpy(), uo) <= 1e-10
    del u
    H = orc.Hierarchy(x.values, x.values)
    ug = cuda.zeros_like(fd)
    uo = np.zeros_like(f)
    mgcycle.v_cycle(h, mgcycle.CycleConfig(smoother="wireframe"), ug, fd)
    orc.v_cycle(H, uo, f, smoother="wireframe", nthreads=nthreads)
    assert _rel(ug.cpu().numpy(), uo) <= 1e-10


@pytest.mark.parametrize("kind", ["zebra_x", "zebra_y"])
def test_zebra_8193_sweep(cuda, orc, kind):
    """Lines of 8191 points exceed one CTA: each runs as a two-legged block
    around its middle point; one sweep against the oracle's line Thomas."""
    n = 8192
    x = grid.make_coords("wall", n, 1.0, 4.0)
    st = stencil.assemble(x, x)
    f = np.zeros((n + 1, n + 1))
    f[1:-1, 1:-1] = Lcg64(9).fill((n - 1, n - 1)) - 0.5
    fd = cuda.from_numpy(f).cuda()
    u = cuda.zeros_like(fd)
    smoothers.sweep(kind, st, smoothers.PlanBundle(n, n), u, fd)
    uo = np.zeros_like(f)
    orc.sweep(kind, (st.W, st.E, st.S, st.N), uo, f, orc.max_threads())
    assert _rel(u.cpu().numpy(), uo) <= 1e-10


@pytest.mark.parametrize("nu", [1, 2])
def test_config3_convergence_factors(cuda, orc, config3, nu):
    """BASELINE config 3, V(1,1) and V(2,2): 20 device cycles at tol=1e-300
    (cli.py:120).  The pre-floor asymptotic factor -- the reference's rule
    (test_acceptance.py:316-322: geometric mean of the cycle ratios, first two
    skipped) with the floor at 1e-7, above the fp64 rounding plateau
     -- over the first 8 cycles matches the oracle's over
    the same cycles to 1e-3, and so do the pre-floor ratios one by one."""
    w, f = config3
    h = grid.build_hierarchy(w.x, w.x)
    cfg = mgcycle.CycleConfig(smoother="tweed", nu1=nu, nu2=nu, tol=1e-300, max_cycles=20)
    _, rep = mgcycle.solve(h, cfg, cuda.from_numpy(f).cuda())
    assert rep.cycles == 20 and all(np.isfinite(rep.defect_norms))
    H = orc.Hierarchy(w.x.values, w.x.values)
    _, repo = orc.solve(H, f, smoother="tweed", nu1=nu, nu2=nu, tol=1e-300, max_cycles=8,
                        nthreads=orc.max_threads())
    assert rep.defect_norms[0] == repo.defect_norms[0]
    # ratios one by one while both relative defects stay above the floor
    # (below it the fp64 rounding of the two summation orders dominates)
    d0 = rep.defect_norms[0]
    pre = 0
    for k, (a, b) in enumerate(zip(rep.per_cycle_ratios[:8], repo.per_cycle_ratios)):
        if min(rep.defect_norms[k + 1], repo.defect_norms[k + 1]) / d0 <= 1e-7:
            break
        assert abs(a - b) <= 1e-3, (k, a, b)
        pre += 1
    assert pre >= 3
    ag = _asymptotic_ratio(rep.defect_norms[:9], floor=1e-7)
    ao = _asymptotic_ratio(repo.defect_norms, floor=1e-7)
    assert abs(ag - ao) <= 1e-3, (ag, ao)
    # the relative defect reaches the rounding floor (~3e-9)
    assert rep.final_rel_defect < 1e-7


@pytest.mark.parametrize("kind", ["tweed", "wireframe"])
def test_exactness_by_colour_large(cuda, kind):
    """After each colour stage the defect vanishes (to rounding) on that
    colour's points, at 2049^2 (test_smoothers.py:54-66 at scale)."""
    from paper_2110_08389_b200 import layout
    n = 2048
    x = grid.make_tanh_wall(n, 1.0, 3.0)
    st = stencil.assemble(x, x)
    rng = np.random.default_rng(7)
    f = np.zeros((n + 1, n + 1))
    f[1:-1, 1:-1] = rng.uniform(-1, 1, (n - 1, n - 1))
    fd = cuda.from_numpy(f).cuda()
    u = cuda.zeros_like(fd)
    ii, jj, _, fl = layout.member_arrays(kind, n, n)
    scale = float(np.max(st.W + st.E) + np.max(st.S + st.N))
    for colour, bit in (("red", 1), ("black", 0)):
        smoothers.sweep_colour(kind, st, u, fd, colour)
        d = stencil.defect(st, u, fd).cpu().numpy()
        sel = (fl & 1) == bit
        worst = np.max(np.abs(d[ii[sel], jj[sel]]))
        umax = float(u.abs().max())
        assert worst <= 1e-12 * scale * max(umax, 1e-300) + 1e-12, (colour, worst)
