"""Look-ahead overlap timeline (dev tool): per depth, ms from the fork to the end of the parent's
inverse (look-ahead stream), to the end of the T GEMM (main stream), and to the join."""
import ctypes, os, sys
sys.path.insert(0, ".")
import torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems, _native
lib = _native.load()
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
inp = solver.prepare(tree, nodes, c.coefficients())
cx = _native.context()
cx.set("profile_ahead", 1)
for it in range(3):
    tl = []
    st = solver.build_device(inp, timeline=tl, stage_begin=lambda name: lib.hps_debug_ahead_depth(cx, 
        int(name.split("_d")[-1]) if name.startswith("merge") else -1))
    torch.cuda.synchronize()
stage = {n: e0.elapsed_time(e1) for n, e0, e1 in tl}
buf = (ctypes.c_float * 3)()
for d in range(2 * c.L):
    if lib.hps_debug_ahead_times(cx, d, buf) == 0:
        print(f"depth {d:2d}: stage {stage[f'merge_d{d}']:.3f} ms | fork -> inverse end {buf[0]:.3f}, T GEMM end {buf[1]:.3f}, join {buf[2]:.3f}")
