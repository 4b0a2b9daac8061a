"""Sharded 3D wireframe V-cycle (BASELINE config 5 across GPUs; SURVEY.md
§8(e)).

CPU: the shell groups (native host functions against numpy), every block in
one group, and multi-process solves over gloo with oracle-backed rank-local
operators, which must equal the single-domain oracle solve bit for bit.
GPU: the same solve on the product path (NativeCubeShardOps) against the
oracle, and partial colour stages against the oracle's partial stages.
"""

import numpy as np
import pytest

from paper_2110_08389_b200 import configs, cube_sharded, sharded

import test_sharded

WORKER = test_sharded.os.path.join(test_sharded.ROOT, "tests", "cube_shard_worker.py")


def _run_workers(tmp_path, world, *args):
    saved = test_sharded.WORKER
    test_sharded.WORKER = WORKER
    try:
        return test_sharded._run_workers(tmp_path, world, *args)
    finally:
        test_sharded.WORKER = saved


def _o3():
    from oracle import oracle3d
    return oracle3d


@pytest.mark.parametrize("scheme", ["wireframe", "tweed"])
@pytest.mark.parametrize("n", [4, 6, 10, 16])
def test_group_sizes_and_offsets(orc, scheme, n):
    gm = _o3().group_map(n, scheme)
    inner = gm[1:-1, 1:-1, 1:-1]
    assert inner.min() >= 1
    sizes = cube_sharded.group_sizes(scheme, n)
    assert (sizes == np.bincount(inner.ravel(), minlength=n // 2 + 1)).all()
    for g0, g1 in [(1, 2), (2, 4), (1, n // 2 + 1), (n // 2, n // 2 + 1)]:
        want = np.flatnonzero((gm >= g0) & (gm < g1))
        assert (cube_sharded.group_offsets(scheme, n, g0, g1) == want).all()


@pytest.mark.parametrize("n", [6, 8, 12])
def test_blocks_lie_in_one_shell(orc, n):
    ii, jj, kk, blk, red = _o3().layout_dump(n, "wireframe")
    gm = _o3().group_map(n, "wireframe")
    g = gm[ii, jj, kk]
    for b in np.unique(blk):
        assert len(np.unique(g[blk == b])) == 1
    # stencil neighbours lie in groups g-1 .. g+1
    inner = gm[1:-1, 1:-1, 1:-1].astype(int)
    for ax in range(3):
        d = np.abs(np.diff(inner, axis=ax))
        assert d.max() <= 1


def test_shell_plan_balances_config5():
    sizes = cube_sharded.group_sizes("wireframe", 1024)
    assert sizes.sum() == 1023 ** 3
    for world in (2, 4, 8):
        b = sharded.balanced_bounds(sizes, world)
        loads = [sizes[b[r]:b[r + 1]].sum() for r in range(world)]
        assert max(loads) / min(loads) < 1.1, loads  # an outer shell is ~5 % of a rank at 8


@pytest.mark.parametrize("n,world", [(16, 2), (32, 2), (48, 3)])
def test_sharded_cube_solve_oracle_ops(orc, tmp_path, n, world):
    outs = _run_workers(tmp_path, world, "--ops", "oracle", "--size", str(n))
    o3 = _o3()
    from paper_2110_08389_b200 import cube
    h = o3.Hierarchy3(configs.sinh_centre(n, 1.0, 3.0).values, scheme="wireframe")
    f = cube.config5_rhs(n, device=False)
    u, rep = o3.solve(h, f, max_cycles=6)
    assert outs[0]["nshard"] >= 1
    for o in outs:
        assert int(o["cycles"]) == rep.cycles
        assert np.array_equal(o["norms"], np.array(rep.defect_norms))
        assert np.array_equal(o["u"], u)


@pytest.mark.gpu
@pytest.mark.parametrize("n,world", [(32, 2), (64, 3)])
def test_sharded_cube_solve_native(orc, cuda, tmp_path, n, world):
    outs = _run_workers(tmp_path, world, "--ops", "native", "--size", str(n))
    o3 = _o3()
    from paper_2110_08389_b200 import cube
    h = o3.Hierarchy3(configs.sinh_centre(n, 1.0, 3.0).values, scheme="wireframe")
    f = cube.config5_rhs(n, device=False)
    u, rep = o3.solve(h, f, max_cycles=6)
    assert outs[0]["nshard"] >= 1
    for o in outs:
        assert int(o["cycles"]) == rep.cycles
        assert np.abs(o["u"] - u).max() <= 1e-10 * np.abs(u).max()
        assert np.array_equal(o["u"], outs[0]["u"])


@pytest.mark.gpu
def test_partial_stages_native(orc, cuda):
    """Colour stages restricted to shell ranges equal the oracle's."""
    import torch
    from paper_2110_08389_b200 import cube
    o3 = _o3()
    n = 32
    x = configs.sinh_centre(n, 1.0, 3.0)
    h = cube.CubeHierarchy(x, scheme="wireframe")
    ops = cube_sharded.NativeCubeShardOps(h)
    st = o3.assemble3(x.values, x.values, x.values)
    rng = np.random.default_rng(11)
    u = np.zeros((n + 1,) * 3)
    u[1:-1, 1:-1, 1:-1] = rng.standard_normal((n - 1,) * 3)
    f = rng.standard_normal((n + 1,) * 3)
    ops.load(torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda())
    uo = u.copy()
    for red, g0, g1 in [(1, 1, 5), (0, 3, 9), (1, 9, 17), (0, 1, 17)]:
        ops.sweep(0, red, g0, g1)
        o3.sweep_part(st, uo, f, red, g0, g1)
    out = torch.empty((n + 1,) * 3, dtype=torch.float64, device="cuda")
    ops.store(out)
    assert np.abs(out.cpu().numpy() - uo).max() <= 1e-12 * np.abs(uo).max()
