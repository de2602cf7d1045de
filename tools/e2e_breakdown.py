"""Host-side breakdown of the end-to-end step (dev tool)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
from paper_1307_2665_b200.grid import layout_of
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
co = c.coefficients()
F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0)
F = F if F.ndim == 2 else F[:, None]
pin_F = torch.from_numpy(np.ascontiguousarray(F)).pin_memory()
U_host = torch.empty((nodes.N, solver.rhs_ld(F.shape[1])), dtype=torch.float64).pin_memory()
lay = layout_of(tree); geom = P.LeafGeometry.get(16, tree.leaf_width, tree.leaf_height)
for it in range(4):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    f = solver._sample(co, lay, geom); t.append(time.perf_counter())
    reps, gid = solver._group(f, 4 ** c.L); t.append(time.perf_counter())
    inp = solver.prepare(tree, nodes, co, pinned=True); torch.cuda.synchronize(); t.append(time.perf_counter())
    st = solver.build_device(inp); t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    Fd = pin_F.to("cuda", non_blocking=True); U = solver.solve_device(st, Fd); torch.cuda.synchronize(); t.append(time.perf_counter())
    U_host.copy_(U, non_blocking=True); solver.check_build(st); torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"sample {d[0]:.1f} group {d[1]:.1f} prepare(total) {d[2]:.1f} build-enqueue {d[3]:.1f} build-gpu-wait {d[4]:.1f} solve {d[5]:.1f} d2h+check {d[6]:.1f} ms")
