"""Debug: V-cycles with / without the black-only prolongation, hybrid / natural layout."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "worker":
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from paper_2110_08389_b200 import grid, mgcycle
    from paper_2110_08389_b200.rng import Lcg64
    out = {}
    for n in (64, 256, 1024, 2048):
        x = grid.make_coords("wall", n, 1.0, 3.0)
        h = grid.build_hierarchy(x, x)
        rng = Lcg64(7)
        f = np.zeros((n + 1, n + 1)); f[1:-1, 1:-1] = rng.fill((n - 1, n - 1)) - 0.5
        u = np.zeros_like(f); u[1:-1, 1:-1] = rng.fill((n - 1, n - 1)) - 0.5
        ud, fd = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
        cfg = mgcycle.CycleConfig(smoother="tweed")
        mgcycle.v_cycle(h, cfg, ud, fd)
        out[str(n)] = ud.cpu().numpy()
    np.savez(sys.argv[2], **out)
    sys.exit(0)
import numpy as np
res = {}
for layout in ("hybrid", "natural"):
    for black in ("0", "1"):
        e = dict(os.environ); e["TMG_PROLONG_BLACK"] = black
        if layout == "natural": e["TMG_LAYOUT"] = "natural"
        path = f"/tmp/dbg_{layout}_{black}.npz"
        r = subprocess.run([sys.executable, __file__, "worker", path], env=e, capture_output=True, text=True)
        if r.returncode: print(r.stderr[-500:])
        z = np.load(path)
        res[(layout, black)] = {int(k): z[k] for k in z.files}
ref = res[("hybrid", "0")]
for key, val in res.items():
    for n in val:
        d = np.abs(val[n] - ref[n]); 
        i, j = np.unravel_index(d.argmax(), d.shape)
        print(key, n, "max rel diff vs hybrid/0: %.3e at (%d,%d)" % (d.max() / np.abs(ref[n]).max(), i, j))
