"""Batched-solve timing for one config (dev tool): median of 10 solves on a built state."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
st = solver.build(tree, nodes, c.coefficients())
F = torch.from_numpy(np.ascontiguousarray(problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0, batch=c.batch))).cuda()
ts = []
for _ in range(12):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); solver.solve_device(st, F); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print(f"cfg{cfg} b={c.batch} solve ms median {np.median(ts[2:]):.3f} min {np.min(ts[2:]):.3f}")
