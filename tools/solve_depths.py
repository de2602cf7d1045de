"""Per-depth timing of the batched solve (dev tool)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems, _native
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
st = solver.build(tree, nodes, c.coefficients())
lib = _native.load()
lay = st.layout
b = c.batch
ldu = solver.rhs_ld(b)
U = torch.zeros((lay.N, ldu), dtype=torch.float64, device="cuda")
res = {}
for rep in range(5):
    for d in range(2 * lay.L):
        dl = lay.depths[d]
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(lib.hps_solve_level(_native.context(), dl.n_boxes, dl.n3, dl.ne, _native.ptr(st.S_levels[d]), _native.ptr(st.Ie_levels[d]),
                                          int(lay.depth_off[d]), _native.ptr(U), ldu, b if b <= 8 else ldu, _native.stream_ptr()), "s")
        e1.record(); e1.synchronize()
        res.setdefault(d, []).append(e0.elapsed_time(e1) * 1e3)
for d in range(2 * lay.L):
    dl = lay.depths[d]
    print(f"  d{d:2d} boxes {dl.n_boxes:5d} n3 {dl.n3:5d} ne {dl.ne:5d}: {np.median(res[d]):8.1f} us")
