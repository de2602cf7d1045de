"""Host coefficient sampling vs chunk count / threads (dev tool)."""
import sys, time, os
sys.path.insert(0, ".")
import numpy as np
import concurrent.futures as cf
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
from paper_1307_2665_b200.grid import layout_of
print("cpus", os.cpu_count())
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 6, 16)
lay = layout_of(tree); geom = P.LeafGeometry.get(16, tree.leaf_width, tree.leaf_height)
co = problems.coefficients(2)
lc = lay.leaf_cells
xs = lay.xline[lc[:, 0]][:, None] + geom.grid_x[None, :]
ys = lay.yline[lc[:, 1]][:, None] + geom.grid_y[None, :]
f = co.c11
t = time.perf_counter(); f(xs, ys); print(f"single call {1e3*(time.perf_counter()-t):.1f} ms")
for nth in (4, 8, 16, 32):
    pool = cf.ThreadPoolExecutor(max_workers=nth)
    for nch in (16, 64, 256):
        b = np.linspace(0, xs.shape[0], nch + 1).astype(int)
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            list(pool.map(lambda ab: f(xs[ab[0]:ab[1]], ys[ab[0]:ab[1]]), zip(b[:-1], b[1:])))
            best = min(best, time.perf_counter() - t)
        print(f"threads {nth:3d} chunks {nch:4d}: {1e3*best:.1f} ms")
    pool.shutdown()
t = time.perf_counter(); solver._sample(co, lay, geom); print(f"_sample (2 fields): {1e3*(time.perf_counter()-t):.1f} ms")
