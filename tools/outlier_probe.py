"""Eager build timing outliers (dev tool): N eager builds of one config with per-stage CUDA events;
prints the stage breakdown of any build more than 20% above the median total."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
inp = solver.prepare(tree, nodes, c.coefficients())
runs = []
for it in range(n):
    tl = []
    t0 = time.perf_counter()
    st = solver.build_device(inp, timeline=tl)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    stages = {nm: e0.elapsed_time(e1) for nm, e0, e1 in tl}
    runs.append((sum(stages.values()), wall * 1e3, stages))
    del st
tot = np.array([r[0] for r in runs])
med = float(np.median(tot))
print(f"median device {med:.3f} ms, min {tot.min():.3f}, max {tot.max():.3f}; wall median {np.median([r[1] for r in runs]):.2f} ms")
for i, (t, w, sg) in enumerate(runs):
    if t > 1.2 * med:
        top = sorted(sg.items(), key=lambda x: -x[1])[:4]
        print(f"  run {i}: {t:.3f} ms (wall {w:.2f}): " + ", ".join(f"{k} {v:.3f}" for k, v in top))
