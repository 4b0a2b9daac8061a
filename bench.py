#!/usr/bin/env python
"""Benchmark of the multigrid V-cycle hot path (BASELINE.json metric:
"smoother grid-pt updates/s; V-cycle time to 1e-10 residual; % HBM roofline").

Default workload (N=1): BASELINE config 3 -- 8193^2 nodes, tanh wall grid
gamma=4, 16-Gaussian RHS (seed 2), tweed smoother, V(2,2), full weighting.
A step is one V(2,2) cycle over the whole hierarchy (13 levels) with u and f
resident in HBM.  value = smoother grid-point updates per second,
(nu1 + nu2) * sum over levels of interior points per cycle / cycle time.

Also reported: the dominant kernel's roofline (one finest-level tweed sweep =
the block-solver launches of both colours, 24 B per interior point
algorithmic), the end-to-end number through the public API with pinned host
buffers copied in and out every step, and the CPU oracle (C restatement of
the reference, 1 core) on one V-cycle of the same workload.

`--impl reference` times the reference algorithm's CPU path (the oracle port,
all host threads) on the same workload and metric.  Under torchrun (N>1) the
one problem is sharded over the ranks (paper_2110_08389_b200.sharded: group
ranges per rank, NCCL halo swaps, replicated coarse tail; strong scaling),
timed on the device and reduced with max over ranks; `--replicas` runs N
independent copies instead (weak scaling).
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0


def _peak_hbm():
    try:
        with open(PEAKS) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = []
        with open(self.path) as fh:
            for r in csv.reader(fh):
                if len(r) >= 9:
                    rows.append([x.strip() for x in r])
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def _updates_per_cycle(h, nu):
    return nu * sum((lv.nx - 1) * (lv.ny - 1) for lv in h.levels)


_DESC = {
    "config1": "tanh wall c=3, f = 2 Lcg64(0) - 1, tweed",
    "config2": "sinh centre gamma=3, f = 2 Lcg64(1) - 1, wireframe",
    "config3": "tanh wall gamma=4, 16 Gaussians (Lcg64(2)), tweed",
    "config4": "tanh wall gamma=3 on all axes, f = 2 Lcg64(3) - 1, 3D tweed",
    "config5": "sinh centre gamma=3 on all axes, f = 2 Lcg64(4) - 1, 3D wireframe",
}


def _config(args, world):
    """The `config` object of the JSON line, identical in both arms (built
    from the arguments only: the reference arm must not import the product
    package)."""
    from oracle import workloads as wl
    n = args.n or wl.CONFIGS[args.config][0]
    dim = 3 if args.config in ("config4", "config5") else 2
    nodes = f"{n + 1}^{dim}"
    nu = args.nu
    upc = wl.updates_per_cycle(n, 2 * nu, dim)
    levels, m = 1, n
    while m % 2 == 0 and m // 2 >= 2:
        levels, m = levels + 1, m // 2
    fb = (n + 1) ** dim * 8
    return {"workload": f"{args.config}: {nodes} nodes fp64, {_DESC[args.config]} "
                        f"V({nu},{nu}), full weighting, {'trilinear' if dim == 3 else 'bilinear'}",
            "levels": levels, "updates_per_cycle": upc,
            "l2": "inputs larger than L2 (u, f = 2 x %.0f MB)" % (fb / 1e6),
            "parallelism": f"{world} rank(s)"}


def asymptotic_ratio(norms, floor=1e-7):
    """Pre-floor asymptotic convergence factor: the reference's rule
    (tests/test_acceptance.py:316-322, geometric mean of the cycle ratios,
    first two skipped) with the floor set above the fp64 rounding plateau
    (SURVEY.md 8(d)): ratios whose new relative defect is <= floor are cut."""
    d = np.asarray(norms, dtype=float)
    if len(d) < 2 or d[0] <= 0:
        return None
    d = d / d[0]
    ratios = [d[k + 1] / d[k] for k in range(len(d) - 1) if d[k + 1] > floor]
    use = ratios[2:] if len(ratios) > 3 else ratios
    return float(np.exp(np.mean(np.log(use)))) if use else None


def run_reference(args):
    """The reference's CPU path (the oracle port, bit-identical to the
    reference's kernels, all host threads) on the same workload.  Imports
    only oracle/ -- never the product package."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import oracle as orc
    from oracle import workloads as wl
    n, x, smoother, rhs = wl.workload(args.config, args.n)
    f = rhs()
    cores = orc.max_threads()
    H = orc.Hierarchy(x, x)
    nu = args.nu

    def cycle():
        u = np.zeros_like(f)
        t0 = time.perf_counter()
        orc.v_cycle(H, u, f, smoother=smoother, nu1=nu, nu2=nu, nthreads=cores)
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        cycle()
    times = [cycle() for _ in range(args.steps)]
    per = float(np.mean(times))
    conf = _config(args, world)
    value = conf["updates_per_cycle"] / per
    sample = f"one V({nu},{nu}) cycle of {args.config} per step, {cores} OpenMP threads"
    line = {
        "impl": "reference", "metric": "smoother grid-pt updates/s", "value": value,
        "unit": "grid-pt updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": conf,
        "cpu_baseline": {"value": value, "unit": "grid-pt updates/s", "cores": cores,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "grid-pt updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    from paper_2110_08389_b200 import _lib, configs, grid, mgcycle
    from paper_2110_08389_b200.stencil import native_level

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    w = configs.workload(args.config, n=args.n, nu=args.nu)
    h = grid.build_hierarchy(w.x, w.x)
    cfg = mgcycle.CycleConfig(smoother=w.smoother, nu1=w.nu1, nu2=w.nu2)
    f_host = w.rhs()
    fd = torch.from_numpy(f_host).cuda()
    u = torch.zeros_like(fd)
    L = _lib.lib()
    state = mgcycle._CycleState(h)
    kind, full, nu1, nu2 = mgcycle._cfg_args(cfg)
    stream = torch.cuda.current_stream()
    import ctypes
    sh = ctypes.c_void_p(stream.cuda_stream)
    up = ctypes.c_void_p(u.data_ptr())
    fp = ctypes.c_void_p(fd.data_ptr())

    # solver session: u and f of the finest level go into the hierarchy's
    # working layout once (outside the timed region); the timed steps are
    # whole V-cycles replayed from a CUDA graph
    _lib.check(L.tmg_session_load(state.native, kind, up, fp, sh))

    def cycles(k):
        _lib.check(L.tmg_session_cycles(state.native, kind, full, nu1, nu2, k, sh))

    for _ in range(max(args.warmup, 3)):
        cycles(1)
    torch.cuda.synchronize()
    for lv in h.levels:
        _lib.check(L.tmg_level_check(native_level(lv.stencil), sh))
    kernels_per_cycle = L.tmg_hier_graph_kernels(state.native)

    clk = ClockSampler(local)
    clk.start()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 1.0:  # clocks settle; sampler covers the timed region
        cycles(20)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = L.tmg_kernel_launches()
    e0.record(stream)
    cycles(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = L.tmg_kernel_launches() - launches0
    t_ms = max_over_ranks(e0.elapsed_time(e1))
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 0.4:
        cycles(20)
        torch.cuda.synchronize()
    clocks = clk.stop()

    # BASELINE metric part 2: the solve (tmg_solve from u = 0, one norm and
    # pivot-flag read-back per cycle).  Configs 1-2: time to a 1e-10
    # relative residual.  Config 3: 20 cycles at tol = 1e-300 and the
    # convergence factor over them (BASELINE config 3; its relative defect
    # floors near 3e-9 in fp64, so 1e-10 is not reachable)
    solve = None
    if not args.no_solve:
        c3 = args.config == "config3"
        tol_s, max_s = (1e-300, 20) if c3 else (1e-10, 50)
        cfg_s = mgcycle.CycleConfig(smoother=w.smoother, nu1=w.nu1, nu2=w.nu2, tol=tol_s,
                                    max_cycles=max_s)
        fd_s = fd.clone()
        mgcycle.solve(h, cfg_s, fd_s)  # warm (plans, graph)
        barrier()
        torch.cuda.synchronize()
        z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        z0.record(stream)
        _, rep = mgcycle.solve(h, cfg_s, fd_s)
        z1.record(stream)
        torch.cuda.synchronize()
        solve = {"tol": tol_s, "max_cycles": max_s, "cycles": rep.cycles,
                 "converged": rep.converged,
                 "ms": max_over_ranks(z0.elapsed_time(z1)),
                 "final_rel_defect": rep.final_rel_defect,
                 "asymptotic_ratio": asymptotic_ratio(rep.defect_norms),
                 "asymptotic_rule": "geometric mean of cycle ratios, first 2 skipped, "
                                    "relative defects <= 1e-7 cut (test_acceptance.py:316-322)"}
        _lib.check(L.tmg_session_load(state.native, kind, up, fp, sh))

    upc = _updates_per_cycle(h, w.nu1 + w.nu2)
    ms_per_step = t_ms / args.steps
    value = world * upc * args.steps / (t_ms * 1e-3)

    # dominant kernel: one finest-level sweep (both colour stages) on the
    # session's working layout, timed alone
    reps = 20
    _lib.check(L.tmg_session_sweeps(state.native, kind, 3, sh))
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    _lib.check(L.tmg_session_sweeps(state.native, kind, reps, sh))
    s1.record(stream)
    torch.cuda.synchronize()
    sweep_ms = s0.elapsed_time(s1) / reps
    n_int = (h.finest.nx - 1) * (h.finest.ny - 1)
    alg_bytes = 24.0 * n_int
    peak, peak_kind = _peak_hbm()
    achieved = alg_bytes / (sweep_ms * 1e-3) / 1e9
    traffic, traffic_src = None, None
    try:  # DRAM bytes of one such sweep from the latest committed ncu capture
        with open(os.path.join(ROOT, "profiles", "latest_traffic.json")) as fh:
            tj = json.load(fh)
        if args.config == "config3" and args.n in (None, 8192):
            traffic = float(tj["bytes_per_sweep"]) / 1e9
            traffic_src = tj.get("source")
    except Exception:
        traffic = None

    # end to end through the public API (mgcycle.v_cycle on CUDA tensors):
    # every step copies its u and f from pinned host memory and reads its u
    # back.  Steps are pipelined over two buffer sets: the H2D copies of step
    # k+1 and the D2H copy of step k-1 run on their own streams (separate
    # copy engines) while step k computes, as a caller streaming problems
    # through the solver would do.  e2e_serial is the same without overlap.
    field_bytes = fd.numel() * 8
    u_h = torch.zeros(fd.shape, dtype=torch.float64).pin_memory()
    f_h = torch.from_numpy(f_host).pin_memory()
    outs = [torch.empty(fd.shape, dtype=torch.float64).pin_memory() for _ in range(2)]
    bufs = [(torch.empty_like(fd), torch.empty_like(fd)) for _ in range(2)]
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()  # noqa: E731
    in_done, cmp_done, out_done = [ev(), ev()], [ev(), ev()], [ev(), ev()]
    e2e_steps = max(2, min(args.steps, 10))

    def pipelined(k_steps):
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for st in (s_in, s_cmp, s_out):
            st.wait_stream(stream)
        for k in range(k_steps):
            b = k % 2
            ue, fe = bufs[b]
            with torch.cuda.stream(s_in):
                if k >= 2:
                    s_in.wait_event(out_done[b])  # buffer b's previous result is out
                fe.copy_(f_h, non_blocking=True)
                ue.copy_(u_h, non_blocking=True)
                in_done[b].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(in_done[b])
                mgcycle.v_cycle(h, cfg, ue, fe, _state=state, check=False)
                cmp_done[b].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(cmp_done[b])
                outs[b].copy_(ue, non_blocking=True)
                out_done[b].record(s_out)
        for st in (s_in, s_cmp, s_out):
            stream.wait_stream(st)
        end.record(stream)
        torch.cuda.synchronize()
        return start.elapsed_time(end)

    def serial(k_steps):
        ue, fe = bufs[0]
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for _ in range(k_steps):
            fe.copy_(f_h, non_blocking=True)
            ue.copy_(u_h, non_blocking=True)
            mgcycle.v_cycle(h, cfg, ue, fe, _state=state, check=False)
            outs[0].copy_(ue, non_blocking=True)
        end.record(stream)
        torch.cuda.synchronize()
        return start.elapsed_time(end)

    pipelined(2)  # warm
    barrier()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(pipelined(e2e_steps)) / e2e_steps
    barrier()
    torch.cuda.synchronize()
    e2e_serial_ms = max_over_ranks(serial(e2e_steps)) / e2e_steps
    e2e = {"value": world * upc / (e2e_ms * 1e-3), "unit": "grid-pt updates/s",
           "h2d_bytes_per_step": 2 * field_bytes, "d2h_bytes_per_step": field_bytes,
           "ms_per_step": e2e_ms, "steps": e2e_steps,
           "mode": "pipelined over 2 buffer sets (H2D / compute / D2H streams)",
           "serial_ms_per_step": e2e_serial_ms,
           "serial_value": world * upc / (e2e_serial_ms * 1e-3)}

    line = {
        "metric": "smoother grid-pt updates/s", "value": value, "unit": "grid-pt updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args, world),
        "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_unit": "GB per launch set",
                     "traffic_source": traffic_src,
                     "kernel": ("leg_sweep_kernel (one finest-level sweep, both colours: "
                                "L-shells, the central cross, the corner points)" if kind == 4 else
                                "block_sweep_kernel (one finest-level sweep, both colours)"),
                     "alg_bytes": alg_bytes, "ms": sweep_ms, "peak_kind": peak_kind},
        "sweep_updates_per_s": n_int / (sweep_ms * 1e-3),
        "solve": solve,
        "e2e": e2e,
        "clocks": clocks,
        "gpu_launches": launches,
        "kernels_per_cycle": kernels_per_cycle,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as orc
        H = orc.Hierarchy(w.x.values, w.x.values)
        uo = np.zeros_like(f_host)
        t0 = time.perf_counter()
        orc.v_cycle(H, uo, f_host, smoother=w.smoother, nu1=w.nu1, nu2=w.nu2, nthreads=1)
        secs = time.perf_counter() - t0
        line["cpu_baseline"] = {
            "value": upc / secs, "unit": "grid-pt updates/s", "cores": 1, "kind": "port",
            "sample": f"one V({w.nu1},{w.nu2}) cycle of the same workload, C oracle, 1 thread "
                      f"({secs:.1f} s)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_sharded(args):
    """N > 1: one problem, fine levels split between the ranks (strong scaling)."""
    import torch
    import torch.distributed as dist

    from paper_2110_08389_b200 import _lib, configs, grid, mgcycle, sharded

    world, rank, local = _dist()
    # TMG_DIST_BACKEND=gloo (halos staged through the host) lets the sharded
    # path be exercised with several ranks on one GPU; timings need nccl
    backend = os.environ.get("TMG_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    L = _lib.lib()
    w = configs.workload(args.config, n=args.n, nu=args.nu)
    h = grid.build_hierarchy(w.x, w.x)
    cfg = mgcycle.CycleConfig(smoother=w.smoother, nu1=w.nu1, nu2=w.nu2)
    f_host = w.rhs()
    fd = torch.from_numpy(f_host).cuda()
    u = torch.zeros_like(fd)
    solver = sharded.ShardedSolver(h, cfg)
    solver.load(u, fd)
    stream = torch.cuda.current_stream()

    def timed(fn, k):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(args.warmup, 3)):
        solver.v_cycle()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    launches0, swaps0 = L.tmg_kernel_launches(), solver.exchanges
    t_ms = timed(solver.v_cycle, args.steps)
    launches = L.tmg_kernel_launches() - launches0
    swaps = (solver.exchanges - swaps0) // args.steps
    clocks = clk.stop()
    upc = _updates_per_cycle(h, w.nu1 + w.nu2)
    value = upc * args.steps / (t_ms * 1e-3)

    # dominant kernel: this rank's finest-level colour stages
    g0, g1 = solver.plan.own(0, rank)
    reps = 20

    def rank_sweep():
        for red in (1, 0):
            solver.ops.sweep(0, red, g0, g1)
    sweep_ms = timed(rank_sweep, reps) / reps
    owned = int(sharded.group_sizes(w.smoother, h.finest.nx, h.finest.ny)[g0:g1].sum())
    alg_bytes = 24.0 * owned
    peak, peak_kind = _peak_hbm()
    achieved = alg_bytes / (sweep_ms * 1e-3) / 1e9

    # end to end: pinned host f and u in, sharded cycle, full u gathered and out
    u_h = torch.zeros(fd.shape, dtype=torch.float64).pin_memory()
    f_h = torch.from_numpy(f_host).pin_memory()
    ue, fe = torch.empty_like(fd), torch.empty_like(fd)

    def e2e_step():
        fe.copy_(f_h, non_blocking=True)
        ue.copy_(u_h, non_blocking=True)
        solver.load(ue, fe)
        solver.v_cycle()
        solver.store(ue)
        u_h.copy_(ue, non_blocking=True)
    e2e_step()
    e2e_steps = max(1, min(args.steps, 5))
    e2e_ms = timed(e2e_step, e2e_steps) / e2e_steps
    field_bytes = fd.numel() * 8
    line = {
        "metric": "smoother grid-pt updates/s", "value": value, "unit": "grid-pt updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args, world),
        "sharded_levels": solver.plan.nshard,
        "parallelism": f"sharded x{world}: group ranges, {backend} halo swaps",
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": "block_sweep_kernel (rank's finest-level share, both colours)",
                     "alg_bytes": alg_bytes, "ms": sweep_ms, "peak_kind": peak_kind},
        "e2e": {"value": upc / (e2e_ms * 1e-3), "unit": "grid-pt updates/s",
                "h2d_bytes_per_step": 2 * field_bytes, "d2h_bytes_per_step": field_bytes,
                "ms_per_step": e2e_ms},
        "clocks": clocks,
        "gpu_launches": launches,
        "halo_swaps_per_cycle": swaps, "dist_backend": backend,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_cube_sharded(args):
    """config 5 with N > 1: one 1025^3 problem, fine levels split between the
    ranks by shells (cube_sharded; strong scaling)."""
    import torch
    import torch.distributed as dist

    from paper_2110_08389_b200 import _lib, cube, cube_sharded, mgcycle

    world, rank, local = _dist()
    backend = os.environ.get("TMG_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    L = _lib.lib()
    n, x = _cube_workload(args)
    h = cube.CubeHierarchy(x, scheme="wireframe")
    cfg = mgcycle.CycleConfig(smoother="wireframe", nu1=2, nu2=2)
    fd = _cube_rhs(args, n)
    u = torch.zeros_like(fd)
    solver = cube_sharded.CubeShardedSolver(h, cfg)
    solver.load(u, fd)
    stream = torch.cuda.current_stream()

    def timed(fn, k):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(args.warmup, 3)):
        solver.v_cycle()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    launches0, swaps0 = L.tmg_kernel_launches(), solver.exchanges
    t_ms = timed(solver.v_cycle, args.steps)
    launches = L.tmg_kernel_launches() - launches0
    swaps = (solver.exchanges - swaps0) // args.steps
    clocks = clk.stop()
    upc = 4 * h.interior_points()
    value = upc * args.steps / (t_ms * 1e-3)
    g0, g1 = solver.plan.own(0, rank)
    reps = 3

    def rank_sweep():
        for red in (1, 0):
            solver.ops.sweep(0, red, g0, g1)
    sweep_ms = timed(rank_sweep, reps) / reps
    owned = int(cube_sharded.group_sizes("wireframe", n)[g0:g1].sum())
    alg_bytes = 24.0 * owned
    peak, peak_kind = _peak_hbm()
    achieved = alg_bytes / (sweep_ms * 1e-3) / 1e9
    u_h = torch.zeros(fd.shape, dtype=torch.float64).pin_memory()
    f_h = fd.cpu().pin_memory()
    ue, fe = torch.empty_like(fd), torch.empty_like(fd)

    def e2e_step():
        fe.copy_(f_h, non_blocking=True)
        ue.copy_(u_h, non_blocking=True)
        solver.load(ue, fe)
        solver.v_cycle()
        solver.store(ue)
        u_h.copy_(ue, non_blocking=True)
    e2e_step()
    e2e_ms = timed(e2e_step, 1)
    field_bytes = fd.numel() * 8
    line = {
        "metric": "smoother grid-pt updates/s", "value": value, "unit": "grid-pt updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args, world),
        "sharded_levels": solver.plan.nshard,
        "parallelism": f"sharded x{world}: shell ranges, {backend} halo swaps",
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": "wblock_kernel (rank's finest-level shells, both colours)",
                     "alg_bytes": alg_bytes, "ms": sweep_ms, "peak_kind": peak_kind},
        "e2e": {"value": upc / (e2e_ms * 1e-3), "unit": "grid-pt updates/s",
                "h2d_bytes_per_step": 2 * field_bytes, "d2h_bytes_per_step": field_bytes,
                "ms_per_step": e2e_ms},
        "clocks": clocks,
        "gpu_launches": launches,
        "halo_swaps_per_cycle": swaps, "dist_backend": backend,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _cube_scheme(args):
    return "wireframe" if args.config == "config5" else "tweed"


def _cube_workload(args):
    from paper_2110_08389_b200 import configs, grid
    if args.config == "config5":
        n = args.n or 1024
        return n, configs.sinh_centre(n, 1.0, 3.0)
    n = args.n or 256
    return n, grid.make_tanh_wall(n, 1.0, 3.0)


def _cube_rhs(args, n, device=True):
    from paper_2110_08389_b200 import cube
    return cube.config5_rhs(n, device) if args.config == "config5" else cube.config4_rhs(n, device)


def run_cube(args):
    """BASELINE config 4 (3D tweed, 257^3) or config 5 (3D wireframe, 1025^3)
    on one GPU (replicas under torchrun)."""
    import ctypes

    import torch

    from paper_2110_08389_b200 import _lib, cube, mgcycle

    world, rank, local = _dist()
    torch.cuda.set_device(local % torch.cuda.device_count())
    n, x = _cube_workload(args)
    scheme = _cube_scheme(args)
    h = cube.CubeHierarchy(x, scheme=scheme)
    f = _cube_rhs(args, n)
    u = torch.zeros_like(f)
    L = _lib.lib()
    stream = torch.cuda.current_stream()
    sh = ctypes.c_void_p(stream.cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    cube._check(L.tmg_cube_load(h._h, P(u), P(f), sh))
    for _ in range(max(args.warmup, 3)):
        cube._check(L.tmg_cube_cycles(h._h, args.nu, args.nu, 1, sh))
    torch.cuda.synchronize()
    clk = ClockSampler(local % torch.cuda.device_count())
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = L.tmg_kernel_launches()
    e0.record(stream)
    cube._check(L.tmg_cube_cycles(h._h, args.nu, args.nu, args.steps, sh))
    e1.record(stream)
    torch.cuda.synchronize()
    launches = L.tmg_kernel_launches() - launches0
    clocks = clk.stop()
    t_ms = e0.elapsed_time(e1)
    upc = 2 * args.nu * h.interior_points()
    value = world * upc * args.steps / (t_ms * 1e-3)
    # dominant kernel: one finest-level 3D sweep
    # convergence factor over a few more cycles of the session (config 5 has
    # no tolerance target: BASELINE quotes V-cycle time)
    out = ctypes.c_double()
    cube._check(L.tmg_cube_norm(h._h, ctypes.byref(out), sh))
    norms = [out.value]
    for _ in range(4):
        cube._check(L.tmg_cube_cycles(h._h, args.nu, args.nu, 1, sh))
        cube._check(L.tmg_cube_norm(h._h, ctypes.byref(out), sh))
        norms.append(out.value)
    ratios = [b / a for a, b in zip(norms, norms[1:]) if a > 0]
    # finest-level sweeps on the session, as the V-cycle runs them (the 3D
    # wireframe on its i- / j-contiguous views; tmg_cube_sweeps ends with one
    # view -> natural conversion, timed alone and subtracted)
    nsw = 10 if n <= 512 else 4

    def timed_sweeps(k):
        cube._check(L.tmg_cube_sweeps(h._h, k, sh))
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        cube._check(L.tmg_cube_sweeps(h._h, k, sh))
        s1.record(stream)
        torch.cuda.synchronize()
        return s0.elapsed_time(s1)
    sweep_ms = (timed_sweeps(nsw) - timed_sweeps(0)) / nsw
    alg = 24.0 * (n - 1) ** 3
    peak, peak_kind = _peak_hbm()
    # end to end: pinned host u, f in; u out; every step (serial)
    u_h = torch.zeros(f.shape, dtype=torch.float64).pin_memory()
    f_h = f.cpu().pin_memory()
    ue, fe = torch.empty_like(f), torch.empty_like(f)
    cfg = mgcycle.CycleConfig(smoother=scheme, nu1=args.nu, nu2=args.nu)

    def e2e_step():
        fe.copy_(f_h, non_blocking=True)
        ue.copy_(u_h, non_blocking=True)
        cube.v_cycle(h, cfg, ue, fe)
        u_h.copy_(ue, non_blocking=True)
    e2e_step()
    torch.cuda.synchronize()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ke = max(1, min(args.steps, 5 if n <= 512 else 2))
    x0.record(stream)
    for _ in range(ke):
        e2e_step()
    x1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = x0.elapsed_time(x1) / ke
    fb = f.numel() * 8
    del ue, fe
    solve = None
    if not args.no_solve and scheme == "tweed":
        cfg_s = mgcycle.CycleConfig(smoother="tweed", nu1=args.nu, nu2=args.nu, tol=1e-10)
        cube.solve(h, cfg_s, f)  # warm (the solve loop's graph), as the 2D solve leg
        torch.cuda.synchronize()
        z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        z0.record(stream)
        _, rep = cube.solve(h, cfg_s, f)
        z1.record(stream)
        torch.cuda.synchronize()
        solve = {"tol": 1e-10, "cycles": rep.cycles, "converged": rep.converged,
                 "ms": z0.elapsed_time(z1), "final_rel_defect": rep.final_rel_defect}
    line = {
        "metric": "smoother grid-pt updates/s", "value": value, "unit": "grid-pt updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args, world),
        "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
        "roofline": {"bound": "hbm", "achieved": alg / (sweep_ms * 1e-3) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": alg / (sweep_ms * 1e-3) / 1e9 / peak,
                     "traffic": None,
                     "kernel": ("wblock_kernel rings + frames, wpoint_kernel (one finest-level 3D "
                                "wireframe sweep)" if scheme == "wireframe" else
                                "wblock_kernel hub blocks + wpoint_kernel (one finest-level 3D tweed sweep)"),
                     "alg_bytes": alg, "ms": sweep_ms, "peak_kind": peak_kind},
        "solve": solve,
        "convergence": {"cycles": len(ratios), "ratios": ratios,
                        "rho": float(np.exp(np.mean(np.log(ratios)))) if ratios else None},
        "e2e": {"value": world * upc / (e2e_ms * 1e-3), "unit": "grid-pt updates/s",
                "h2d_bytes_per_step": 2 * fb, "d2h_bytes_per_step": fb, "ms_per_step": e2e_ms},
        "clocks": clocks,
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle3d as o3
        if n <= 256:
            H = o3.Hierarchy3(x.values, scheme=scheme)
            fh = f.cpu().numpy()
            uo = np.zeros_like(fh)
            t0 = time.perf_counter()
            o3.v_cycle(H, uo, fh, args.nu, args.nu, 1)
            secs = time.perf_counter() - t0
            sample = (f"one V({args.nu},{args.nu}) cycle of the same workload, 3D C oracle, "
                      f"1 thread ({secs:.1f} s)")
            cpu_v = upc / secs
        else:  # bounded sample: >= 10 s of sweeps of the 257^3 cube of the same grid family
            n_s = 256
            xs = x.values[:: n // n_s].copy()
            fs = np.ascontiguousarray(f[:: n // n_s, :: n // n_s, :: n // n_s].cpu().numpy())
            us = np.zeros_like(fs)
            st = o3.assemble3(xs, xs, xs)
            nsw, t0 = 0, time.perf_counter()
            while nsw == 0 or time.perf_counter() - t0 < 10.0:
                o3.sweep(st, us, fs, 1, scheme)
                nsw += 1
            secs = time.perf_counter() - t0
            cpu_v = nsw * (n_s - 1) ** 3 / secs
            sample = (f"{nsw} 3D {scheme} sweeps of a 257^3 cube (every {n // n_s}th node of "
                      f"the same grid), C oracle, 1 thread ({secs:.1f} s)")
        line["cpu_baseline"] = {"value": cpu_v, "unit": "grid-pt updates/s", "cores": 1,
                                "kind": "port", "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_cube_reference(args):
    """Configs 4-5 through the 3D C oracle with all host threads; imports
    only oracle/ (never the product package)."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import oracle as orc
    from oracle import oracle3d as o3
    from oracle import workloads as wl
    n, x, scheme, rhs = wl.workload(args.config, args.n)
    cores = orc.max_threads()
    conf = _config(args, world)
    times = []
    f = rhs()
    if n <= 256:  # one V-cycle of the workload per step
        H = o3.Hierarchy3(x, scheme=scheme)
        steps, warm = args.steps, args.warmup
        for k in range(warm + steps):
            u = np.zeros_like(f)
            t0 = time.perf_counter()
            o3.v_cycle(H, u, f, args.nu, args.nu, cores)
            if k >= warm:
                times.append(time.perf_counter() - t0)
        per = float(np.mean(times))
        value = conf["updates_per_cycle"] / per
        sample = f"one V({args.nu},{args.nu}) cycle per step, 3D C oracle, {cores} OpenMP threads"
    else:  # bounded: one finest-level sweep of the full grid per step (<= 3 steps)
        st = o3.assemble3(x, x, x)
        u = np.zeros_like(f)
        steps, warm = min(args.steps, 3), 1
        for k in range(warm + steps):
            t0 = time.perf_counter()
            o3.sweep(st, u, f, cores, scheme)
            if k >= warm:
                times.append(time.perf_counter() - t0)
        per = float(np.mean(times))
        value = (n - 1) ** 3 / per
        sample = (f"one finest-level 3D {scheme} sweep of the {n + 1}^3 workload per step "
                  f"({steps} steps after {warm} warm-up), C oracle, {cores} OpenMP threads")
    line = {
        "impl": "reference", "metric": "smoother grid-pt updates/s", "value": value,
        "unit": "grid-pt updates/s", "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": conf,
        "cpu_baseline": {"value": value, "unit": "grid-pt updates/s", "cores": cores,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "grid-pt updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--config", default="config3",
                   choices=("config1", "config2", "config3", "config4", "config5"))
    p.add_argument("--intervals", "--n", dest="n", type=int, default=None,
                   help="override grid intervals (use --intervals under torchrun)")
    p.add_argument("--nu", type=int, default=2, help="config3: V(nu,nu)")
    p.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    p.add_argument("--no-solve", action="store_true", help="skip the time-to-1e-10 solve")
    p.add_argument("--replicas", action="store_true",
                   help="N > 1: independent replicas instead of one sharded problem")
    args = p.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.config in ("config4", "config5"):
        if args.impl == "reference":
            run_cube_reference(args)
        elif args.config == "config5" and _dist()[0] > 1 and not args.replicas:
            run_cube_sharded(args)
        else:
            run_cube(args)
    elif args.impl == "reference":
        run_reference(args)
    elif _dist()[0] > 1 and not args.replicas:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
