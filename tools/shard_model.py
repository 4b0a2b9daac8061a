"""Per-rank compute of the sharded V(2,2) cycle, measured on ONE B200 with
the exchanges stubbed out, plus a model of the halo / all-gather traffic, for
DESIGN.md §7.  Not a scaling measurement: every gpurun box has one GPU.

For world W and each rank r of the config-3 plan, the rank's whole cycle
(its partial sweeps, partial transfers, halo gather / scatter kernels, the
replicated tail) is timed with CUDA events; the exchange calls return at
once and the all-gather hands back a buffer of the right size.  The model
adds, per swap, a latency t_lat and bytes / B_link, and per all-gather the
gathered bytes / B_link.

usage: python tools/shard_model.py [W ...]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2110_08389_b200 import configs, grid, mgcycle, sharded


class StubComm:
    def __init__(self, rank, world):
        self.rank, self.world, self.backend = rank, world, "stub"
        self.swaps = 0
        self.swap_bytes = 0
        self.gather_bytes = 0

    def exchange(self, pairs):
        self.swaps += 1
        self.swap_bytes += sum(int(s.numel()) * 8 for _, s, _ in pairs)

    def allgather(self, t, counts):
        self.gather_bytes += 8 * (sum(counts) - int(t.numel()))
        return torch.zeros(sum(counts), dtype=t.dtype, device=t.device)

    def allreduce_max(self, vals, device):
        return list(vals)


def main():
    worlds = [int(a) for a in sys.argv[1:]] or [2, 4, 8]
    w = configs.workload("config3")
    h = grid.build_hierarchy(w.x, w.x)
    f = torch.from_numpy(w.rhs()).cuda()
    u = torch.zeros_like(f)
    cfg = mgcycle.CycleConfig(smoother="tweed", nu1=2, nu2=2)
    t_lat, b_link = 10e-6, 700e9  # per p2p swap (s), NVLink 5 per direction (B/s)
    out = {}
    for W in worlds:
        per_rank = []
        only = os.environ.get("SHARD_RANK")
        for r in ([int(only)] if only is not None else range(W)):
            comm = StubComm(r, W)
            solver = sharded.ShardedSolver(h, cfg, comm=comm)
            solver.load(u, f)
            solver.v_cycle()  # warm-up (plans, kernels)
            torch.cuda.synchronize()
            sw0, sb0, gb0 = comm.swaps, comm.swap_bytes, comm.gather_bytes
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            a.record()
            for _ in range(reps):
                solver.v_cycle()
            b.record()
            torch.cuda.synchronize()
            ms_eager = a.elapsed_time(b) / reps
            # the same rank cycle captured in a CUDA graph (the device work
            # alone, no Python / launch gaps between the ~500 operations)
            g = torch.cuda.CUDAGraph()
            s_ = torch.cuda.Stream()
            s_.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_):
                solver.v_cycle()
            torch.cuda.current_stream().wait_stream(s_)
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                solver.v_cycle()
            g.replay()
            torch.cuda.synchronize()
            a.record()
            for _ in range(reps):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            calls = reps + 2  # eager reps, the warm-up before capture, the capture
            swaps = (comm.swaps - sw0) / calls
            sbytes = (comm.swap_bytes - sb0) / calls
            gbytes = (comm.gather_bytes - gb0) / calls
            model_ms = ms + 1e3 * (swaps * t_lat + sbytes / b_link + gbytes / b_link)
            per_rank.append({"rank": r, "compute_ms": ms, "eager_ms": ms_eager, "swaps": swaps,
                             "swap_MB": sbytes / 1e6, "gather_MB": gbytes / 1e6,
                             "modelled_ms": model_ms, "nshard": solver.plan.nshard})
            del solver
            torch.cuda.empty_cache()
        worst = max(per_rank, key=lambda d: d["modelled_ms"])
        out[W] = {"ranks": per_rank, "cycle_ms_modelled": worst["modelled_ms"],
                  "compute_ms_max": max(d["compute_ms"] for d in per_rank)}
        print(json.dumps({"world": W, "compute_ms_max": out[W]["compute_ms_max"],
                          "cycle_ms_modelled": out[W]["cycle_ms_modelled"],
                          "swaps": worst["swaps"], "nshard": worst["nshard"]}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
