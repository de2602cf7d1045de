import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
from _util import rel
for cfg, L in ((3, 7), (3, 6), (1, 7)):
    t0 = time.time()
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
    st = solver.build(tree, nodes, problems.coefficients(cfg))
    F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=4, batch=1)
    u = solver.solve(st, F)
    ex = problems.exact_solution(cfg, nodes.points[:, 0], nodes.points[:, 1], seed=4, batch=1)
    L1 = st.geometry.L1; Ie = st.layout.leaf_I_e
    e = rel(np.einsum("rc,lc->lr", L1, u[Ie]), np.einsum("rc,lc->lr", L1, ex[Ie]))
    print(f"cfg{cfg} L={L} exact L1u rel err {e:.2e} ({time.time()-t0:.1f} s)", flush=True)
t0 = time.time()
cfg, L = 5, 9
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
st = solver.build(tree, nodes, problems.coefficients(cfg))
T = st.root_T.device_tensor
one = torch.ones(T.shape[0], dtype=torch.float64, device=T.device)
print("cfg5 L=9 constants in DtN null space:", float((T @ one).abs().max() / T.abs().max()), f"({time.time()-t0:.1f} s)", flush=True)
F = problems.boundary_data(2, nodes.points[tree.root.I_e], seed=9, batch=2)
u = solver.solve(st, F)
uc = solver.solve(st, 2.0 * F[:, 0] - 3.0 * F[:, 1])
L1 = st.geometry.L1; Ie = st.layout.leaf_I_e
lin = np.einsum("rc,lc->lr", L1, 2.0 * u[Ie, 0] - 3.0 * u[Ie, 1])
print("cfg5 L=9 linearity:", rel(np.einsum("rc,lc->lr", L1, uc[Ie]), lin), f"({time.time()-t0:.1f} s)", flush=True)
