"""Do timing events recorded inside a captured build work on replay? (dev tool)"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
c = problems.CONFIGS[2]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
inp = solver.prepare(tree, nodes, c.coefficients())
st = solver.build_device(inp); torch.cuda.synchronize(); del st
g = torch.cuda.CUDAGraph()
tl = []
try:
    with torch.cuda.graph(g):
        st = solver.build_device(inp, timeline=tl)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    print("captured markers:", len(tl), [(n, round(a.elapsed_time(b), 3)) for n, a, b in tl[:4]])
except Exception as e:
    print("capture with events failed:", type(e).__name__, str(e)[:300])
