"""3D wireframe on cubes (BASELINE config 5).  There is no 3D reference
(SURVEY.md §8(c)); the CPU restatement oracle/wire3d_oracle.c is pinned by
property tests here (partition, block shapes, same-colour independence,
agreement with a dense block Gauss-Seidel, convergence), and the device path
is checked against it."""

import numpy as np
import pytest

from paper_2110_08389_b200 import configs, grid

from test_3d import _dense


def _o3():
    from oracle import oracle3d
    return oracle3d


@pytest.mark.parametrize("n", [4, 6, 8, 12, 16])
def test_layout_partition_and_colouring(orc, n):
    o3 = _o3()
    ii, jj, kk, blk, red = o3.layout_dump(n, "wireframe")
    pts = list(zip(ii.tolist(), jj.tolist(), kk.tolist()))
    assert len(set(pts)) == len(pts) == (n - 1) ** 3
    owner = {p: (b, r) for p, b, r in zip(pts, blk.tolist(), red.tolist())}
    for p, (bl, r) in owner.items():
        for d in ((1, 0, 0), (0, 1, 0), (0, 0, 1)):
            q = (p[0] + d[0], p[1] + d[1], p[2] + d[2])
            if q in owner and owner[q][0] != bl:
                assert owner[q][1] != r, (p, q)
    # the corners and every frame are red
    assert owner[(1, 1, 1)][1] == 1


@pytest.mark.parametrize("n", [6, 8, 12])
def test_block_shapes(orc, n):
    """Every block is a frame (8 corners of degree 3, 12 paths), a closed
    ring (every member has exactly two in-block neighbours) or a point."""
    o3 = _o3()
    ii, jj, kk, blk, red = o3.layout_dump(n, "wireframe")
    members = {}
    for p, b in zip(zip(ii.tolist(), jj.tolist(), kk.tolist()), blk.tolist()):
        members.setdefault(b, set()).add(p)
    c = n // 2
    kinds = {"frame": 0, "ring": 0, "point": 0}
    for b, pts in members.items():
        deg = {}
        for p in pts:
            deg[p] = sum((p[0] + d0, p[1] + d1, p[2] + d2) in pts
                         for d0, d1, d2 in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0),
                                            (0, 0, 1), (0, 0, -1)))
        if len(pts) == 1:
            kinds["point"] += 1
        elif sorted(deg.values()).count(3) == 8:
            assert set(deg.values()) == {2, 3}
            r = min(min(p) for p in pts)
            assert len(pts) == 8 + 12 * (n - 2 * r - 1)
            kinds["frame"] += 1
        else:
            assert set(deg.values()) == {2}, b
            kinds["ring"] += 1
    assert kinds["frame"] == c - 1
    assert kinds["ring"] == 6 * sum(c - 1 - s for s in range(1, c))
    assert kinds["point"] == 1 + 6 * (c - 1)


@pytest.mark.parametrize("n", [4, 6, 8])
def test_sweep_equals_dense_block_gauss_seidel(orc, n):
    o3 = _o3()
    x = configs.sinh_centre(n, 1.0, 3.0).values
    st = o3.assemble3(x, x, x)
    rng = np.random.default_rng(7)
    u = np.zeros((n + 1,) * 3)
    u[1:-1, 1:-1, 1:-1] = rng.standard_normal((n - 1,) * 3)
    f = rng.standard_normal((n + 1,) * 3)
    uo = u.copy()
    o3.sweep(st, uo, f, scheme="wireframe")
    A, idx = _dense(st, n)
    ii, jj, kk, blk, red = o3.layout_dump(n, "wireframe")
    v = u[1:-1, 1:-1, 1:-1].reshape(-1).copy()
    fv = f[1:-1, 1:-1, 1:-1].reshape(-1)
    for colour in (1, 0):
        for b in np.unique(blk[red == colour]):
            sel = blk == b
            I = np.array([idx(a, bb, c) for a, bb, c in zip(ii[sel], jj[sel], kk[sel])])
            mask = np.ones(len(v), bool)
            mask[I] = False
            v[I] = np.linalg.solve(A[np.ix_(I, I)], fv[I] - A[np.ix_(I, mask)] @ v[mask])
    assert np.abs(uo[1:-1, 1:-1, 1:-1].reshape(-1) - v).max() <= 1e-12 * np.abs(v).max()


def test_oracle_vcycle_converges(orc):
    o3 = _o3()
    n = 16
    h = o3.Hierarchy3(configs.sinh_centre(n, 1.0, 3.0).values, scheme="wireframe")
    f = np.zeros((n + 1,) * 3)
    f[1:-1, 1:-1, 1:-1] = np.random.default_rng(4).uniform(-1, 1, (n - 1,) * 3)
    _, rep = o3.solve(h, f, max_cycles=40)
    assert rep.converged
    assert max(rep.per_cycle_ratios[2:]) < 0.5


# ----------------------------------------------------------------------------
# device path against the oracle

@pytest.mark.gpu
@pytest.mark.parametrize("n", [4, 6, 8, 16, 32, 66, 130])
def test_device_sweep_matches_oracle(cuda, orc, n):
    from paper_2110_08389_b200 import cube
    o3 = _o3()
    x = configs.sinh_centre(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x, scheme="wireframe")
    rng = np.random.default_rng(5)
    u = np.zeros((n + 1,) * 3)
    u[1:-1, 1:-1, 1:-1] = rng.standard_normal((n - 1,) * 3)
    f = rng.standard_normal((n + 1,) * 3)
    ug = u.copy()
    cube.sweep(h, ug, f)
    uo = u.copy()
    o3.sweep(o3.assemble3(x.values, x.values, x.values), uo, f, scheme="wireframe")
    assert np.abs(ug - uo).max() <= 1e-12 * np.abs(uo).max()
    assert np.all(ug[0] == 0) and np.all(ug[:, :, -1] == 0)


@pytest.mark.gpu
def test_device_vcycle_and_solve_match_oracle(cuda, orc):
    from paper_2110_08389_b200 import cube, mgcycle
    o3 = _o3()
    n = 32
    x = configs.sinh_centre(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x, scheme="wireframe")
    H = o3.Hierarchy3(x.values, scheme="wireframe")
    f = cube.config5_rhs(n, device=False)
    cfg = mgcycle.CycleConfig(smoother="wireframe", nu1=2, nu2=2)
    ug, uo = np.zeros_like(f), np.zeros_like(f)
    for _ in range(2):
        cube.v_cycle(h, cfg, ug, f)
        o3.v_cycle(H, uo, f)
        assert np.abs(ug - uo).max() <= 1e-10 * np.abs(uo).max()
    _, rep = cube.solve(h, cfg, f)
    _, repo = o3.solve(H, f)
    assert rep.cycles == repo.cycles and rep.converged == repo.converged
    for a, b in zip(rep.defect_norms, repo.defect_norms):
        assert abs(a - b) <= 1e-6 * b + 1e-11 * repo.defect_norms[0]


@pytest.mark.gpu
def test_config5_scale_sweep(cuda, orc):
    """513^3 (half the config-5 grid, so the oracle finishes in seconds): one
    device sweep against the oracle."""
    from paper_2110_08389_b200 import cube
    o3 = _o3()
    n = 512
    x = configs.sinh_centre(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x, scheme="wireframe")
    f = cube.config5_rhs(n)
    u = cube.config5_rhs(n) * 0.5
    uo = u.cpu().numpy()
    cube.sweep(h, u, f)
    o3.sweep(o3.assemble3(x.values, x.values, x.values), uo, f.cpu().numpy(), orc.max_threads(),
             scheme="wireframe")
    assert np.abs(u.cpu().numpy() - uo).max() <= 1e-10 * np.abs(uo).max()


@pytest.mark.gpu
def test_config5_full_size_sweep_and_cycle(cuda, orc):
    """BASELINE config 5 at its full 1025^3 size (the 64-thread-edge PCR
    path and the 16-point chunks only occur here): one finest-level sweep on
    the API layout and one V(2,2) cycle (hybrid views, every level) against
    the oracle with all host threads, gate 1e-10."""
    import gc

    from paper_2110_08389_b200 import cube, mgcycle
    o3 = _o3()
    n = 1024
    nthreads = orc.max_threads()
    x = configs.sinh_centre(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x, scheme="wireframe")
    f = cube.config5_rhs(n, device=False)
    fd = cuda.from_numpy(f).cuda()
    u = cuda.zeros_like(fd)
    cube.sweep(h, u, fd)
    uo = np.zeros_like(f)
    o3.sweep(o3.assemble3(x.values, x.values, x.values), uo, f, nthreads, scheme="wireframe")
    got = u.cpu().numpy()
    assert np.abs(got - uo).max() <= 1e-10 * np.abs(uo).max()
    del got, u
    gc.collect()
    ug = cuda.zeros_like(fd)
    cube.v_cycle(h, mgcycle.CycleConfig(smoother="wireframe", nu1=2, nu2=2), ug, fd)
    uo[...] = 0.0
    H = o3.Hierarchy3(x.values, scheme="wireframe")
    o3.v_cycle(H, uo, f, 2, 2, nthreads)
    got = ug.cpu().numpy()
    assert np.abs(got - uo).max() <= 1e-10 * np.abs(uo).max()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [16, 32])
def test_hybrid_vcycle_matches_oracle(cuda, orc, monkeypatch, n):
    """The V-cycle on the hybrid layout (i- and j-contiguous views of every
    level, forced down to n = 4) against the oracle, per cycle and in the
    solve's cycle count."""
    from paper_2110_08389_b200 import cube, mgcycle
    monkeypatch.setenv("TMG_HYB_MIN", "4")
    o3 = _o3()
    x = configs.sinh_centre(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x, scheme="wireframe")
    H = o3.Hierarchy3(x.values, scheme="wireframe")
    f = cube.config5_rhs(n, device=False)
    cfg = mgcycle.CycleConfig(smoother="wireframe", nu1=2, nu2=2)
    ug, uo = np.zeros_like(f), np.zeros_like(f)
    for _ in range(3):
        cube.v_cycle(h, cfg, ug, f)
        o3.v_cycle(H, uo, f)
        assert np.abs(ug - uo).max() <= 1e-10 * np.abs(uo).max()
    _, rep = cube.solve(h, cfg, f)
    _, repo = o3.solve(H, f)
    assert rep.cycles == repo.cycles and rep.converged == repo.converged


@pytest.mark.gpu
@pytest.mark.parametrize("te", [32, 64])
@pytest.mark.parametrize("hyb", ["4", "100000"])
def test_wide_classes_match_oracle(cuda, orc, monkeypatch, te, hyb):
    """Rings and frames forced into the wide launch classes (TE threads per
    edge: 64 spans two warps, the PCR path of the 1025^3 cube) on a small
    cube, natural and hybrid, against the oracle."""
    from paper_2110_08389_b200 import cube, mgcycle
    monkeypatch.setenv("TMG_FORCE_TE", str(te))
    monkeypatch.setenv("TMG_HYB_MIN", hyb)
    o3 = _o3()
    n = 32
    x = configs.sinh_centre(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x, scheme="wireframe")
    rng = np.random.default_rng(9)
    u = np.zeros((n + 1,) * 3)
    u[1:-1, 1:-1, 1:-1] = rng.standard_normal((n - 1,) * 3)
    f = rng.standard_normal((n + 1,) * 3)
    ug, uo = u.copy(), u.copy()
    cube.sweep(h, ug, f)
    o3.sweep(o3.assemble3(x.values, x.values, x.values), uo, f, scheme="wireframe")
    assert np.abs(ug - uo).max() <= 1e-12 * np.abs(uo).max()
    H = o3.Hierarchy3(x.values, scheme="wireframe")
    fc = cube.config5_rhs(n, device=False)
    cfg = mgcycle.CycleConfig(smoother="wireframe", nu1=2, nu2=2)
    ug, uo = np.zeros_like(fc), np.zeros_like(fc)
    for _ in range(2):
        cube.v_cycle(h, cfg, ug, fc)
        o3.v_cycle(H, uo, fc)
        assert np.abs(ug - uo).max() <= 1e-10 * np.abs(uo).max()


@pytest.mark.gpu
def test_cube_argument_errors(cuda):
    """Shape, scheme and size errors map to ValueError (the C ABI's
    TMG_BADARG), before any device work."""
    from paper_2110_08389_b200 import cube, mgcycle
    x = configs.sinh_centre(8, 1.0, 3.0)
    with pytest.raises(ValueError):
        cube.CubeHierarchy(configs.sinh_centre(7, 1.0, 3.0), scheme="wireframe")
    with pytest.raises(ValueError):
        cube.CubeHierarchy(x, scheme="checkerboard")
    with pytest.raises(ValueError):  # rings longer than 64 threads x 16 points
        cube.CubeHierarchy(np.linspace(0.0, 1.0, 1031), scheme="wireframe")
    h = cube.CubeHierarchy(x, scheme="wireframe")
    with pytest.raises(ValueError):
        cube.sweep(h, np.zeros((8, 9, 9)), np.zeros((9, 9, 9)))
    with pytest.raises(ValueError):
        cube.v_cycle(h, mgcycle.CycleConfig(smoother="tweed"), np.zeros((9,) * 3), np.zeros((9,) * 3))


@pytest.mark.gpu
def test_sweeps_entry_matches_single_sweeps(cuda, orc):
    """tmg_cube_sweeps (session sweeps on the hybrid views, forced here) equals
    repeated natural sweeps of the same fields."""
    import ctypes
    import os
    import torch
    from paper_2110_08389_b200 import _lib, cube
    n = 32
    x = configs.sinh_centre(n, 1.0, 3.0)
    os.environ["TMG_HYB_MIN"] = "4"
    try:
        h = cube.CubeHierarchy(x, scheme="wireframe")
    finally:
        del os.environ["TMG_HYB_MIN"]
    rng = np.random.default_rng(3)
    u0 = np.zeros((n + 1,) * 3)
    u0[1:-1, 1:-1, 1:-1] = rng.standard_normal((n - 1,) * 3)
    f = rng.standard_normal((n + 1,) * 3)
    ud, fd = torch.from_numpy(u0).cuda(), torch.from_numpy(f).cuda()
    L, s = _lib.lib(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    cube._check(L.tmg_cube_load(h._h, ctypes.c_void_p(ud.data_ptr()), ctypes.c_void_p(fd.data_ptr()), s))
    cube._check(L.tmg_cube_sweeps(h._h, 3, s))
    out = torch.empty_like(ud)
    cube._check(L.tmg_cube_store(h._h, ctypes.c_void_p(out.data_ptr()), s))
    ref = u0.copy()
    for _ in range(3):
        cube.sweep(h, ref, f)
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.gpu
def test_config5_full_size_properties(cuda):
    """BASELINE config 5 at its full 1025^3 size, where the CPU oracle is too
    slow to run in a test, through size-independent properties: the session's
    hybrid-view sweep equals the natural-layout sweep (1e-12), one sweep is
    affine in f (S(u, f1 + f2) - S(u, f1) = S(0, f2) - S(0, 0), S(0, 0) = 0 on
    the homogeneous Dirichlet cube), and V(2,2) cycles reduce the defect at
    the factor the bench reports (rho < 0.9)."""
    import ctypes
    import torch
    from paper_2110_08389_b200 import _lib, cube
    n = 1024
    x = configs.sinh_centre(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x, scheme="wireframe")
    L, s = _lib.lib(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    f1 = cube.config5_rhs(n)
    f2 = torch.roll(f1, shifts=(3, 5, 7), dims=(0, 1, 2)) * 0.5
    f2[0], f2[-1], f2[:, 0], f2[:, -1], f2[:, :, 0], f2[:, :, -1] = 0, 0, 0, 0, 0, 0
    u = f1 * 0.25
    # hybrid session sweep vs natural sweep
    cube._check(L.tmg_cube_load(h._h, P(u), P(f1), s))
    cube._check(L.tmg_cube_sweeps(h._h, 1, s))
    hyb = torch.empty_like(u)
    cube._check(L.tmg_cube_store(h._h, P(hyb), s))
    nat = u.clone()
    cube._check(L.tmg_cube_sweep(h._h, P(nat), P(f1), s))
    scale = nat.abs().max().item()
    assert (hyb - nat).abs().max().item() <= 1e-12 * scale
    del hyb
    # affine in f
    a = u.clone()
    cube._check(L.tmg_cube_sweep(h._h, P(a), P(f1 + f2), s))
    a -= nat
    del nat
    b = torch.zeros_like(u)
    cube._check(L.tmg_cube_sweep(h._h, P(b), P(f2), s))
    # a is a difference of O(scale) sweeps: rounding relative to their size
    assert (a - b).abs().max().item() <= 1e-12 * scale
    del a, b
    # convergence of the hybrid V-cycle
    z = torch.zeros_like(u)
    cube._check(L.tmg_cube_load(h._h, P(z), P(f1), s))
    out = ctypes.c_double()
    cube._check(L.tmg_cube_norm(h._h, ctypes.byref(out), s))
    norms = [out.value]
    for _ in range(3):
        cube._check(L.tmg_cube_cycles(h._h, 2, 2, 1, s))
        cube._check(L.tmg_cube_norm(h._h, ctypes.byref(out), s))
        norms.append(out.value)
    ratios = [q / p for p, q in zip(norms, norms[1:])]
    assert all(r < 0.9 for r in ratios), ratios
