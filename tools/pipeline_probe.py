"""Timeline of solver.Pipeline over many jobs (dev tool): prepare start/end per job, yield times."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nj = int(sys.argv[2]) if len(sys.argv) > 2 else 12
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
co = c.coefficients()
F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0, batch=c.batch)
F = torch.from_numpy(np.ascontiguousarray(F if F.ndim == 2 else F[:, None])).pin_memory()
pipe = solver.Pipeline(tree, nodes, reuse_graphs=len(sys.argv) > 3)
T0 = [0.0]
log = []
orig = pipe._prepare
def timed_prepare(coeffs):
    a = time.perf_counter()
    r = orig(coeffs)
    log.append(("prep", a - T0[0], time.perf_counter() - T0[0]))
    return r
pipe._prepare = timed_prepare
for rep in range(2):
    log.clear()
    torch.cuda.synchronize()
    T0[0] = time.perf_counter()
    for U, st in pipe.run([(co, F)] * nj):
        log.append(("yield", time.perf_counter() - T0[0], 0))
        st = None
    torch.cuda.synchronize()
    tot = time.perf_counter() - T0[0]
print(f"{nj} jobs: {1e3*tot:.1f} ms total, {1e3*tot/nj:.2f} ms/job")
for k, a, b in log:
    print(f"  {k:5s} {1e3*a:8.2f} {1e3*b:8.2f}" if k == "prep" else f"  {k:5s} {1e3*a:8.2f}")
pipe.overlap_results = False
for rep in range(2):
    log.clear()
    torch.cuda.synchronize()
    T0[0] = time.perf_counter()
    for U, st in pipe.run([(co, F)] * nj):
        log.append(("yield", time.perf_counter() - T0[0], 0))
        st = None
    torch.cuda.synchronize()
    tot = time.perf_counter() - T0[0]
print(f"no result overlap: {nj} jobs: {1e3*tot:.1f} ms total, {1e3*tot/nj:.2f} ms/job")
for k, a, b in log:
    print(f"  {k:5s} {1e3*a:8.2f} {1e3*b:8.2f}" if k == "prep" else f"  {k:5s} {1e3*a:8.2f}")
