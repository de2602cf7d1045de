"""Per-stage CUDA-event breakdown of build + solve for one config (dev tool)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
from paper_1307_2665_b200 import work as O
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
L = int(sys.argv[2]) if len(sys.argv) > 2 else problems.CONFIGS[cfg].L
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
for it in range(3):
    tl = []
    torch.cuda.synchronize(); t0 = time.time()
    st = solver.build(tree, nodes, c.coefficients(), timeline=tl)
    torch.cuda.synchronize(); t1 = time.time()
print(f"cfg{cfg} L={L} wall build {t1-t0:.4f}s groups {st.n_leaf_groups}")
tot = 0
for name, e0, e1 in tl:
    ms = e0.elapsed_time(e1); tot += ms
    if name == "leaf":
        fl = st.n_leaf_groups * O.leaf_flops(16)
    else:
        d = int(name.split("d")[1]); n3, ne = O.depth_sizes(L, 16, d)
        fl = (2 ** d) * (2/3*n3**3 + 2*n3*n3*ne + 2*n3*ne*ne)
    print(f"  {name:10s} {ms:8.3f} ms  {fl/ms/1e9:8.2f} TF/s(alg)")
print(f"  device total {tot:.3f} ms")
F = torch.from_numpy(problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0)).cuda()
for it in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); U = solver.solve_device(st, F); e1.record(); e1.synchronize()
print(f"  solve b={F.shape[1] if F.dim()>1 else 1}: {e0.elapsed_time(e1):.3f} ms")
