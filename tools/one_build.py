"""Build (and solve) one config once after a small warm-up: target for ncu launch lists."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
L = int(sys.argv[2]) if len(sys.argv) > 2 else problems.CONFIGS[cfg].L
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
st = solver.build(tree, nodes, c.coefficients())
F = torch.from_numpy(problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0)).cuda()
U = solver.solve_device(st, F)
torch.cuda.synchronize()
print("ok")
