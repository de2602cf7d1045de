import sys, os
import os; _here = os.path.dirname(os.path.abspath(__file__)); sys.path.insert(0, os.path.dirname(_here)); sys.path.insert(0, _here)
import numpy as np
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems
from oracle import hps_oracle as O
from _util import coeff_dict, rel
for (q, L, cfg) in ((12, 5, 4), (12, 4, 4), (21, 4, 4), (16, 5, 4)):
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, q)
    st = solver.build(tree, nodes, problems.coefficients(cfg), check=False)
    ot = O.build_tree((0, 1, 0, 1), L, q)
    ost = O.build(ot, coeff_dict(problems.coefficients(cfg)))
    F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=1, batch=12)
    u = solver.solve(st, F)
    print(os.environ.get("HPS_AHEAD_MIN_N3", "default"), q, L, cfg, "rootT", f"{rel(st.root_T.dense, ost.root_T):.2e}",
          "L1u", f"{rel(O.leaf_cheb_boundary(ost, u), O.leaf_cheb_boundary(ost, O.solve(ost, F))):.2e}", flush=True)
