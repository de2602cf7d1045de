"""Small post_process run for compute-sanitizer (dev tool)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 2, 16)
st = solver.build(tree, nodes, problems.coefficients(2))
f = problems.boundary_data(2, nodes.points[tree.root.I_e], seed=3, batch=1)
u = solver.solve(st, f)
W = solver.leaf_fields(st, u)
torch.cuda.synchronize()
print("fields ok", W.shape)
print(solver.post_process(st, u, [(0.13, 0.71), (0.5, 0.5)]))
