"""One config-1 V(2,2) cycle through the public API (for the TMG_MINI_TIMING
build's per-phase clock printout of the shared-memory tail)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08389_b200 import configs, grid, mgcycle

w = configs.workload(sys.argv[1] if len(sys.argv) > 1 else "config1")
h = grid.build_hierarchy(w.x, w.x)
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
cfg = mgcycle.CycleConfig(smoother=w.smoother, nu1=2, nu2=2)
for _ in range(3):
    mgcycle.v_cycle(h, cfg, u, f)
torch.cuda.synchronize()
print("done")
