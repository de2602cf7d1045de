"""Print the SPEC acceptance-criteria numbers (E_pot, E_grad, E_int, leaf-DtN convergence) (dev tool)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, scipy.special
import test_gpu_spec as T
from paper_1307_2665_b200 import solver
from paper_1307_2665_b200.leafops import CoefficientField
tree, nodes = T._tree(4)
st = solver.build(tree, nodes, CoefficientField())
gam = nodes.points[tree.root.I_e]
u = solver.solve(st, T._log(gam))
ug = solver.gauge_fixed_solution(st, u).cpu().numpy()
inner = T._interior(nodes, tree)
e_pot = np.max(np.abs(ug[inner] - T._log(nodes.points)[inner]))
e_raw = np.max(np.abs(u[inner] - T._log(nodes.points)[inner]))
v = solver.apply_global_dtn(st, T._log(gam))
e_grad = np.max(np.abs(v - T._coord_flux(nodes, tree, *T._log_grad(gam))))
print(f"criterion 1/3 (Laplace log, L=4): E_pot {e_pot:.2e} (raw Gauss u {e_raw:.2e}), E_grad {e_grad:.2e}, ratio {e_grad/e_pot:.0f}")
kappa = 40.0
st = solver.build(tree, nodes, CoefficientField(c=-kappa ** 2))
ex = lambda p: scipy.special.y0(kappa * np.hypot(p[:, 0] + 2.0, p[:, 1]))
ug = solver.gauge_fixed_solution(st, solver.solve(st, ex(gam))).cpu().numpy()
print(f"criterion 2 (Helmholtz Y0, kappa 40, L=4): E_pot {np.max(np.abs(ug[inner] - ex(nodes.points)[inner])):.2e}")
co = CoefficientField(c1=-1000.0, c2=-1000.0)
f = lambda p: np.sin(np.pi * p[:, 0]) + np.cos(2.0 * p[:, 1]) + p[:, 0] * p[:, 1]
vals = []
for L in (2, 3, 4, 5):
    tr, nd = T._tree(L)
    s = solver.build(tr, nd, co)
    vals.append(float(solver.post_process(s, solver.solve(s, f(nd.points[tr.root.I_e])), np.array([[0.75, 0.25]]))[0]))
print("criterion 8 (conv-diff -1000): E_int(L=2,3,4) =", ", ".join(f"{e:.2e}" for e in np.abs(np.diff(vals))))
errs = []
for q in (6, 8, 10, 12, 14, 16):
    tr, nd = T._tree(0, q)
    s = solver.build(tr, nd, CoefficientField())
    g = nd.points[tr.root.I_e]
    errs.append(np.max(np.abs(solver.apply_global_dtn(s, T._log(g)) - T._coord_flux(nd, tr, *T._log_grad(g)))))
print("criterion 9 (leaf DtN, q=6..16): ", ", ".join(f"{e:.2e}" for e in errs))
