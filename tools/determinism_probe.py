"""Build the same config twice eagerly and report the first stage whose output differs (dev tool)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
for cfg in [int(a) for a in sys.argv[1:]] or [3]:
    c = problems.CONFIGS[cfg]
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
    inp = solver.prepare(tree, nodes, c.coefficients())
    runs = []
    for r in range(3):
        st = solver.build_device(inp, keep_level_T=True)
        torch.cuda.synchronize()
        runs.append(st)
    a, b, cc = runs
    print(f"cfg{cfg}: c12 nonzero? {getattr(c, 'name', '')}")
    for name in ("root_T",):
        print(" root_T equal 0-1", torch.equal(a.root_T.device_tensor, b.root_T.device_tensor),
              "0-2", torch.equal(a.root_T.device_tensor, cc.root_T.device_tensor))
    for attr in dir(a):
        pass
    print("  leaf T equal", torch.equal(a.T_leaf_groups, b.T_leaf_groups), "psi equal", torch.equal(a.psi_groups, b.psi_groups))
    for d in range(len(a.S_levels) - 1, -1, -1):
        x, y = a.level_T[d], b.level_T[d]
        if x is None:
            continue
        print(f"  depth {d}: T equal={torch.equal(x, y)} maxdiff={float((x-y).abs().max()):.3e}  S equal={torch.equal(a.S_levels[d], b.S_levels[d])}")
