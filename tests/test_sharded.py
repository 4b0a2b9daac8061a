"""Sharded V-cycle.

CPU: the group decomposition (native host functions against the oracle's
restatement), the partition and halo bookkeeping, and full multi-process
solves over gloo with oracle-backed rank-local operators, which must equal
the single-domain oracle solve bit for bit.
GPU: the same multi-process solve on the product path (the sm_100a library
behind NativeShardOps, halos staged through gloo) against the oracle, plus
partial sweeps against the oracle's partial sweeps.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2110_08389_b200 import sharded

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "shard_worker.py")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_workers(tmp_path, world, *args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", WORKER, "--out", str(tmp_path), *args]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [dict(np.load(tmp_path / f"rank{k}.npz")) for k in range(world)]


def _oracle_solve(orc, kind, n, ny=None, restriction="full", max_cycles=50):
    from paper_2110_08389_b200 import grid, mgcycle
    ny = ny or n
    x, y = grid.make_coords("wall", n, 1.0, 3.0), grid.make_coords("wall", ny, 2.0, 2.0)
    oh = orc.Hierarchy(x.values, y.values)
    f = mgcycle.random_rhs(n, ny, 7)
    return orc.solve(oh, f, smoother=kind, restriction=restriction, max_cycles=max_cycles)


# ---------------------------------------------------------------------------
# group decomposition

@pytest.mark.parametrize("kind", sharded.SHARDABLE)
@pytest.mark.parametrize("nx,ny", [(16, 16), (32, 16), (16, 40), (64, 64)])
def test_group_sizes_match_oracle(orc, kind, nx, ny):
    gm = orc.group_map(kind, nx, ny)
    want = np.bincount(gm[1:-1, 1:-1].ravel(), minlength=gm.max() + 1)
    got = sharded.group_sizes(kind, nx, ny)
    assert len(got) == sharded.group_count(kind, nx, ny) + 1
    assert np.array_equal(got, want)


@pytest.mark.parametrize("kind", sharded.SHARDABLE)
def test_blocks_lie_in_one_group(orc, kind):
    """Every block of the reference layout lies inside one group, and the
    groups of a block's stencil neighbours differ by at most one."""
    nx, ny = 24, 16
    gm = orc.group_map(kind, nx, ny)
    if kind != "checkerboard":
        ii, jj, blk, _ = orc.layout_dump(kind, nx, ny)
        for b in np.unique(blk):
            sel = blk == b
            assert len(np.unique(gm[ii[sel], jj[sel]])) == 1
    inner = gm[1:-1, 1:-1]
    assert np.abs(np.diff(inner, axis=0)).max() <= 1
    assert np.abs(np.diff(inner, axis=1)).max() <= 1


@pytest.mark.parametrize("kind", sharded.SHARDABLE)
def test_coarse_group_is_half(orc, kind):
    gf, gc = orc.group_map(kind, 32, 32), orc.group_map(kind, 16, 16)
    assert np.array_equal(gf[2:-2:2, 2:-2:2], 2 * gc[1:-1, 1:-1])


@pytest.mark.parametrize("kind", sharded.SHARDABLE)
def test_group_offsets_decode(orc, kind):
    """Encoded positions address each point of the groups once, in the
    session layout of the kind (N buffer C order, T buffer transposed)."""
    nx, ny = 20, 16
    gm = orc.group_map(kind, nx, ny)
    enc = sharded.group_offsets(kind, nx, ny, 3, 7)
    off, tb = enc >> 1, enc & 1
    i = np.where(tb == 1, off % (nx + 1), off // (ny + 1))
    j = np.where(tb == 1, off // (nx + 1), off % (ny + 1))
    assert np.all((gm[i, j] >= 3) & (gm[i, j] < 7))
    assert len(enc) == np.count_nonzero((gm >= 3) & (gm < 7))
    assert len(set(zip(i.tolist(), j.tolist()))) == len(enc)


# ---------------------------------------------------------------------------
# partition bookkeeping

def test_balanced_bounds():
    sizes = np.array([0] + [8 * k for k in range(1, 101)])
    b = sharded.balanced_bounds(sizes, 4)
    assert b[0] == 1 and b[-1] == 101 and all(b[k] < b[k + 1] for k in range(4))
    loads = [sizes[b[k]:b[k + 1]].sum() for k in range(4)]
    assert max(loads) / min(loads) < 1.1
    with pytest.raises(ValueError):
        sharded.balanced_bounds(np.array([0, 1, 1]), 3)


def test_coarse_bounds_nest():
    b = [1, 40, 71, 101]
    cb = sharded.coarse_bounds(b, 50)
    assert cb[0] == 1 and cb[-1] == 51
    for r in range(3):  # coarse G owned by the owner of fine 2G
        for G in range(cb[r], cb[r + 1]):
            assert b[r] <= 2 * G < b[r + 1]


def test_shard_plan_levels():
    dims = [(1024 >> k, 1024 >> k) for k in range(10)]
    p = sharded.ShardPlan.build("tweed", dims, 4, sizes_fn=sharded.group_sizes)
    assert 1 <= p.nshard < len(dims)
    assert len(p.bounds) == p.nshard + 1
    for lvl in range(p.nshard):
        assert min(np.diff(p.bounds[lvl])) >= 4
    h0 = p.halo(0, 1)
    assert [peer for peer, _, _ in h0] == [0, 2]
    (_, snd, rcv), _ = h0
    assert snd == (p.bounds[0][1], p.bounds[0][1] + 2) and rcv == (p.bounds[0][1] - 2,
                                                                  p.bounds[0][1])
    assert sharded.ShardPlan.build("tweed", dims, 1).nshard == 0
    with pytest.raises(ValueError):
        sharded.ShardPlan.build("zebra_alt", dims, 2)


# ---------------------------------------------------------------------------
# multi-process solves (gloo)

@pytest.mark.parametrize("kind,n,ny,world,restriction", [
    ("tweed", 64, 64, 2, "full"),
    ("wireframe", 64, 64, 2, "full"),
    ("tweed", 64, 32, 3, "full"),
    ("tweed", 128, 128, 4, "half"),
    ("zebra_x", 32, 32, 2, "full"),
    ("zebra_y", 32, 48, 3, "half"),
    ("checkerboard", 32, 32, 2, "full"),
])
def test_sharded_solve_oracle_ops(orc, tmp_path, kind, n, ny, world, restriction):
    """world ranks over gloo with oracle rank-local operators reproduce the
    single-domain oracle solve bit for bit (same cycles, same norms, same u)."""
    u_ref, rep = _oracle_solve(orc, kind, n, ny, restriction=restriction, max_cycles=12)
    outs = _run_workers(tmp_path, world, "--ops", "oracle", "--kind", kind, "--nx", str(n),
                        "--ny", str(ny), "--max-cycles", "12", "--min-groups", "3",
                        "--restriction", restriction)
    for o in outs:
        assert int(o["nshard"]) >= 1
        assert int(o["cycles"]) == rep.cycles
        assert np.array_equal(o["norms"], np.array(rep.defect_norms))
        assert np.array_equal(o["u"], u_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n,world", [("tweed", 256, 2), ("wireframe", 128, 2),
                                          ("zebra_x", 64, 2), ("checkerboard", 64, 2),
                                          ("tweed", 256, 4), ("wireframe", 256, 4)])
def test_sharded_solve_native(orc, cuda, tmp_path, kind, n, world):
    """The product path sharded over ranks equals the single-domain oracle
    (per-sweep 1e-10 north-star tolerance on the final iterate; identical
    cycle counts)."""
    u_ref, rep = _oracle_solve(orc, kind, n, max_cycles=12)
    outs = _run_workers(tmp_path, world, "--ops", "native", "--kind", kind, "--nx", str(n),
                        "--max-cycles", "12")
    for o in outs:
        assert int(o["nshard"]) >= 1
        assert int(o["cycles"]) == rep.cycles
        d0 = rep.defect_norms[0]
        for a, b in zip(o["norms"], rep.defect_norms):
            assert abs(a - b) <= 1e-5 * b + 1e-11 * d0
        scale = np.abs(u_ref).max()
        assert np.abs(o["u"] - u_ref).max() <= 1e-10 * scale
    for o in outs[1:]:
        assert np.array_equal(outs[0]["u"], o["u"])


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n", [(k, 64) for k in sharded.SHARDABLE] +
                         [("tweed", 600), ("tweed", 1026)])
def test_partial_sweeps_native(orc, cuda, kind, n):
    """Colour stages over group ranges on the device equal the oracle's
    partial stages; the ranges together equal one full sweep.  At n >= 1024
    the tweed ranges run their L-shells (and, in the last range, the cross)
    on the leg kernel."""
    import torch

    from paper_2110_08389_b200 import _device, _lib, grid, mgcycle
    x, y = grid.make_coords("wall", n, 1.0, 3.0), grid.make_coords("wall", n, 2.0, 2.0)
    h = grid.build_hierarchy(x, y)
    st = h.finest.stencil
    sto = tuple(np.asarray(a) for a in (st.W, st.E, st.S, st.N))
    rng = np.random.default_rng(3)
    u0 = np.zeros((n + 1, n + 1))
    u0[1:-1, 1:-1] = rng.standard_normal((n - 1, n - 1))
    f = mgcycle.random_rhs(n, n, 5)
    G = sharded.group_count(kind, n, n)
    cuts = [1, G // 3, G // 2 + 1, G + 1]
    ops = sharded.NativeShardOps(h, kind)
    ud, fd = _device.to_device(u0), _device.to_device(f)
    ops.load(ud, fd)
    uo = u0.copy()
    for red in (1, 0):
        for a, b in zip(cuts[:-1], cuts[1:]):
            ops.sweep(0, red, a, b)
            orc.sweep_part(kind, sto, uo, f, red, a, b)
    out = torch.zeros_like(ud)
    ops.store(out)
    got = out.cpu().numpy()
    ufull = u0.copy()
    orc.sweep(kind, sto, ufull, f)
    assert np.array_equal(uo, ufull)
    assert np.abs(got - uo).max() <= 1e-12 * np.abs(uo).max()
    _lib.check(_lib.lib().tmg_session_check(ops.native, _device.stream_handle()))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", sharded.SHARDABLE)
def test_partial_transfers_native(orc, cuda, kind):
    """One rank's share of the transfers (tmg_session_restrict_part /
    _prolong_part): restricting group range by group range, then prolonging
    range by range, gives bit for bit the full-level transfers, and the
    coarse u is zeroed exactly on the requested groups."""
    import ctypes

    import torch

    from paper_2110_08389_b200 import _device, _lib, grid

    n, m = 300, 260
    x, y = grid.make_coords("wall", n, 1.0, 3.0), grid.make_coords("centre", m, 1.0, 1.5)
    h = grid.build_hierarchy(x, y)
    rng = np.random.default_rng(11)
    u0 = rng.standard_normal((n + 1, m + 1))
    f = rng.standard_normal((n + 1, m + 1))
    L = _lib.lib()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    kid = _lib.KIND_IDS[kind]
    nc, mc = n // 2, m // 2

    def run(parts):
        ops = sharded.NativeShardOps(h, kind)
        ops.load(_device.to_device(u0), _device.to_device(f))
        fill = torch.full((nc + 1, mc + 1), 7.0, dtype=torch.float64, device="cuda")
        if parts is None:
            ops.restrict(0)
        else:
            for g in parts:
                ops.restrict(0, g)
        fc = torch.empty_like(fill)
        uc = torch.empty_like(fill)
        _lib.check(L.tmg_session_read(ops.native, 1, 1, P(fc), s))
        _lib.check(L.tmg_session_read(ops.native, 1, 0, P(uc), s))
        # a nonzero coarse correction, then the prolongation (tensors kept
        # alive: the caching allocator would hand a freed block straight on)
        enc = ops.offsets(1, 1, Gc + 1)
        vals = torch.linspace(-1, 1, int(enc.numel()), dtype=torch.float64, device="cuda")
        _lib.check(L.tmg_session_scatter(ops.native, 1, 0, P(enc), int(enc.numel()), P(vals), s))
        if parts is None:
            ops.prolong(0)
        else:
            for g in fparts:
                ops.prolong(0, g)
        out = torch.empty((n + 1, m + 1), dtype=torch.float64, device="cuda")
        ops.store(out)
        torch.cuda.synchronize()
        return fc.cpu().numpy(), uc.cpu().numpy(), out.cpu().numpy()

    Gc = sharded.group_count(kind, nc, mc)
    G = sharded.group_count(kind, n, m)
    cparts = [(1, Gc // 3), (Gc // 3, Gc // 2 + 1), (Gc // 2 + 1, Gc + 1)]
    fparts = [(1, G // 4), (G // 4, G // 2), (G // 2, G + 1)]
    fa, ua, oa = run(None)
    fb, ub, ob = run(cparts)
    assert np.array_equal(fa[1:-1, 1:-1], fb[1:-1, 1:-1])
    assert not ub[1:-1, 1:-1].any()
    assert np.array_equal(oa, ob)
    # the coarse points outside a partial range keep their values
    fc1, uc1, _ = run([cparts[0]])
    gm = orc.group_map(kind, nc, mc)
    inside = (gm >= cparts[0][0]) & (gm < cparts[0][1])
    assert np.array_equal(fc1[inside], fa[inside])
