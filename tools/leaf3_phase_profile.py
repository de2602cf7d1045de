"""Per-phase cycle breakdown of k_leaf16v3 (tools/libhps_b200_prof.so built with -DHPS_LEAF_PROFILE)."""
import os, sys, ctypes
os.environ.setdefault("HPS_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhps_b200_prof.so"))
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems, _native
lib = _native.load()
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
L = problems.CONFIGS[cfg].L
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
inp = solver.prepare(tree, nodes, problems.coefficients(cfg))
solver.build_device(inp); torch.cuda.synchronize()
buf = (ctypes.c_longlong * (1024 * 16))()
lib.hps_debug_leaf3_profile(buf, 1)
tl = []
solver.build_device(inp, timeline=tl); torch.cuda.synchronize()
lib.hps_debug_leaf3_profile(buf, 0)
a = np.frombuffer(buf, dtype=np.int64).reshape(1024, 16)[:296].astype(float)
per = inp.ngroups / 296
names = ["assembly", "factor(0)", "U12 (13x)", "U-warps: lookahead cols", "U-warps: total update", "P-warps: wait for lookahead",
         "P-warps: wait+factor", "panel iteration total", "back substitution", "epilogue", "BS: Y staging", "BS: wait at block barrier", "BS: tri-solve (warp 0)", "BS: update (warp 0)"]
print("leaf ms", [round(e0.elapsed_time(e1), 3) for n, e0, e1 in tl if n == "leaf"])
for i, n in enumerate(names):
    print(f"  {n:30s} {a[:, i].mean() / per:12.0f} cyc/leaf")
