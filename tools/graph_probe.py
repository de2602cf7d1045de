"""Eager build+solve vs CUDA-graph replay of the same sequence (dev experiment)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
inp = solver.prepare(tree, nodes, c.coefficients())
F = torch.from_numpy(np.ascontiguousarray(problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0))).cuda()
if F.dim() == 1: F = F[:, None]
def step():
    st = solver.build_device(inp)
    U = solver.solve_device(st, F)
    return st, U
for _ in range(3): step()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record(); step(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print("eager ms", np.round(ts, 3))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()  # warm-up on the side stream
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    st_g, U_g = step()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0.record(); g.replay(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print("graph ms", np.round(ts, 3))
st_e, U_e = step(); torch.cuda.synchronize()
print("graph vs eager max |dU|", float((U_g - U_e).abs().max()), "root T equal", bool(torch.equal(st_g.root_T.device_tensor, st_e.root_T.device_tensor)))
