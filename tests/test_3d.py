"""3D tweed on cubes (BASELINE config 4).  There is no 3D reference
(SURVEY.md §8(c)); the CPU restatement oracle/tweed3d_oracle.c is pinned by
property tests here (partition, same-colour independence, agreement with a
dense block Gauss-Seidel, convergence), and the device path is checked
against it."""

import numpy as np
import pytest

from paper_2110_08389_b200 import grid


def _o3():
    from oracle import oracle3d
    return oracle3d


def _dense(st, n):
    W, E, S, N, B, T = st
    m = (n - 1) ** 3
    A = np.zeros((m, m))

    def idx(i, j, k):
        return ((i - 1) * (n - 1) + (j - 1)) * (n - 1) + (k - 1)

    for i in range(1, n):
        for j in range(1, n):
            for k in range(1, n):
                r = idx(i, j, k)
                A[r, r] = -(W[i] + E[i] + S[j] + N[j] + B[k] + T[k])
                for di, dj, dk, c in ((-1, 0, 0, W[i]), (1, 0, 0, E[i]), (0, -1, 0, S[j]),
                                      (0, 1, 0, N[j]), (0, 0, -1, B[k]), (0, 0, 1, T[k])):
                    a, b, cc = i + di, j + dj, k + dk
                    if 1 <= a < n and 1 <= b < n and 1 <= cc < n:
                        A[r, idx(a, b, cc)] = c
    return A, idx


@pytest.mark.parametrize("n", [4, 6, 8, 12])
def test_layout_partition_and_colouring(orc, n):
    o3 = _o3()
    ii, jj, kk, blk, red = o3.layout_dump(n)
    assert len(set(zip(ii.tolist(), jj.tolist(), kk.tolist()))) == len(ii) == (n - 1) ** 3
    owner = {}
    for a, b, c, bl, r in zip(ii.tolist(), jj.tolist(), kk.tolist(), blk.tolist(), red.tolist()):
        owner[(a, b, c)] = (bl, r)
    for p, (bl, r) in owner.items():
        for d in ((1, 0, 0), (0, 1, 0), (0, 0, 1)):
            q = (p[0] + d[0], p[1] + d[1], p[2] + d[2])
            if q in owner and owner[q][0] != bl:
                assert owner[q][1] != r, (p, q)
    # corners are red; every block is a tree of straight legs into its branch
    assert owner[(1, 1, 1)][1] == 1


@pytest.mark.parametrize("n", [4, 6, 8])
def test_sweep_equals_dense_block_gauss_seidel(orc, n):
    o3 = _o3()
    x = grid.make_tanh_wall(n, 1.0, 2.0).values
    st = o3.assemble3(x, x, x)
    rng = np.random.default_rng(1)
    u = np.zeros((n + 1,) * 3)
    u[1:-1, 1:-1, 1:-1] = rng.standard_normal((n - 1,) * 3)
    f = rng.standard_normal((n + 1,) * 3)
    uo = u.copy()
    o3.sweep(st, uo, f)
    A, idx = _dense(st, n)
    ii, jj, kk, blk, red = o3.layout_dump(n)
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
    h = o3.Hierarchy3(grid.make_tanh_wall(n, 1.0, 3.0).values)
    f = np.zeros((n + 1,) * 3)
    f[1:-1, 1:-1, 1:-1] = np.random.default_rng(3).uniform(-1, 1, (n - 1,) * 3)
    _, rep = o3.solve(h, f, max_cycles=30)
    assert rep.converged and rep.cycles <= 15
    assert max(rep.per_cycle_ratios[2:]) < 0.2


# ----------------------------------------------------------------------------
# device path against the oracle

@pytest.mark.gpu
@pytest.mark.parametrize("n", [4, 8, 16, 32])
def test_device_sweep_matches_oracle(cuda, orc, n):
    from paper_2110_08389_b200 import cube
    o3 = _o3()
    x = grid.make_tanh_wall(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x)
    rng = np.random.default_rng(5)
    u = np.zeros((n + 1,) * 3)
    u[1:-1, 1:-1, 1:-1] = rng.standard_normal((n - 1,) * 3)
    f = rng.standard_normal((n + 1,) * 3)
    ug = u.copy()
    cube.sweep(h, ug, f)
    uo = u.copy()
    o3.sweep(o3.assemble3(x.values, x.values, x.values), uo, f)
    assert np.abs(ug - uo).max() <= 1e-12 * np.abs(uo).max()
    # boundary untouched
    assert np.all(ug[0] == 0) and np.all(ug[:, :, -1] == 0)


@pytest.mark.gpu
def test_device_defect_bit_identical(cuda, orc):
    from paper_2110_08389_b200 import cube
    o3 = _o3()
    n = 16
    x = grid.make_tanh_wall(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x)
    rng = np.random.default_rng(2)
    u = rng.standard_normal((n + 1,) * 3)
    f = rng.standard_normal((n + 1,) * 3)
    assert np.array_equal(cube.defect(h, u, f),
                          o3.defect(o3.assemble3(x.values, x.values, x.values), u, f))


@pytest.mark.gpu
def test_device_vcycle_and_solve_match_oracle(cuda, orc):
    from paper_2110_08389_b200 import cube, mgcycle
    o3 = _o3()
    n = 32
    x = grid.make_tanh_wall(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x)
    H = o3.Hierarchy3(x.values)
    f = cube.config4_rhs(n, device=False)
    cfg = mgcycle.CycleConfig(smoother="tweed", nu1=2, nu2=2)
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
def test_device_lcg_rhs_matches_host(cuda):
    from paper_2110_08389_b200 import cube
    n = 24
    assert np.array_equal(cube.config4_rhs(n).cpu().numpy(), cube.config4_rhs(n, device=False))


@pytest.mark.gpu
def test_config4_scale_sweep(cuda, orc):
    """257^3 (BASELINE config 4 grid): one device sweep against the oracle."""
    from paper_2110_08389_b200 import cube
    o3 = _o3()
    n = 256
    x = grid.make_tanh_wall(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x)
    f = cube.config4_rhs(n)
    u = cube.config4_rhs(n) * 0.5
    uo = u.cpu().numpy()
    cube.sweep(h, u, f)
    o3.sweep(o3.assemble3(x.values, x.values, x.values), uo, f.cpu().numpy(), orc.max_threads())
    assert np.abs(u.cpu().numpy() - uo).max() <= 1e-10 * np.abs(uo).max()


@pytest.mark.gpu
def test_hybrid_vcycle_matches_oracle(cuda, orc, monkeypatch):
    """3D tweed V-cycle on the hybrid layout (leg-axis views, forced down to
    n = 4) against the oracle."""
    from paper_2110_08389_b200 import cube, mgcycle
    monkeypatch.setenv("TMG_HYB_MIN", "4")
    o3 = _o3()
    n = 32
    x = grid.make_tanh_wall(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x)
    H = o3.Hierarchy3(x.values)
    f = cube.config4_rhs(n, device=False)
    cfg = mgcycle.CycleConfig(smoother="tweed", nu1=2, nu2=2)
    ug, uo = np.zeros_like(f), np.zeros_like(f)
    for _ in range(3):
        cube.v_cycle(h, cfg, ug, f)
        o3.v_cycle(H, uo, f)
        assert np.abs(ug - uo).max() <= 1e-10 * np.abs(uo).max()


@pytest.mark.gpu
@pytest.mark.parametrize("te", [16, 32])
def test_wide_hub_classes_match_oracle(cuda, orc, monkeypatch, te):
    """3D tweed hub blocks forced into the wide launch classes (TE threads
    per leg, as on the 1025^3 cube) on a small cube, natural and hybrid,
    against the oracle."""
    from paper_2110_08389_b200 import cube, mgcycle
    monkeypatch.setenv("TMG_FORCE_TE", str(te))
    o3 = _o3()
    n = 32
    x = grid.make_tanh_wall(n, 1.0, 3.0)
    for hyb in ("4", "100000"):
        monkeypatch.setenv("TMG_HYB_MIN", hyb)
        h = cube.CubeHierarchy(x)
        H = o3.Hierarchy3(x.values)
        f = cube.config4_rhs(n, device=False)
        cfg = mgcycle.CycleConfig(smoother="tweed", nu1=2, nu2=2)
        ug, uo = np.zeros_like(f), np.zeros_like(f)
        for _ in range(2):
            cube.v_cycle(h, cfg, ug, f)
            o3.v_cycle(H, uo, f)
            assert np.abs(ug - uo).max() <= 1e-10 * np.abs(uo).max()
