"""Phase clocks of the leg kernel (needs the -DTMG_LEGK_TIMING library:
make -C paper_2110_08389_b200/csrc timing; run with
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_timing.so TMG_LEGK_TIMING=1)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08389_b200 import _lib, configs, grid, mgcycle

w = configs.workload("config3")
h = grid.build_hierarchy(w.x, w.x)
f = torch.from_numpy(w.rhs()).cuda()
u = torch.zeros_like(f)
L = _lib.lib()
st = mgcycle._CycleState(h)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
_lib.check(L.tmg_session_load(st.native, 4, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), s))
_lib.check(L.tmg_session_sweeps(st.native, 4, 2, s))
torch.cuda.synchronize()
# last launch = the black stage of the finest level's second sweep
out = (ctypes.c_double * 24)()
n = L.tmg_debug_leg_phases(out)
names = ["setup", "wait", "forward", "back", "reduced", "branch", "finalize", "loadissue",
         "storeissue", "blobwait", "storeread", "-"]
for who, vals in (("thread0", list(out)[:12]), ("thread96", list(out)[12:])):
    tot = sum(vals)
    print(json.dumps({"who": who, "ctas": n, "cycles_per_cta": tot,
                      "share": {k: round(v / tot, 3) for k, v in zip(names, vals)}}))

ids = (ctypes.c_int * 1024)()
k = L.tmg_debug_leg_smids(ids, 1024)
pairs = [(ids[2 * c], ids[2 * c + 1]) for c in range(k // 2)]
same = sum(1 for a, b in pairs if a == b)
from collections import Counter
per_sm = Counter(ids[i] for i in range(k))
print(json.dumps({"clusters": len(pairs), "pairs_on_one_sm": same,
                  "ctas_per_sm": dict(Counter(per_sm.values()))}))
