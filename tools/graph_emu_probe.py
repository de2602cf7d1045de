import sys, warnings, torch, numpy as np
sys.path.insert(0, ".")
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems, _native
warnings.simplefilter("always")
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 7, 16)
inp = solver.prepare(tree, nodes, problems.coefficients(5))
F = torch.from_numpy(problems.boundary_data(5, nodes.points[tree.root.I_e], seed=0, batch=8)).cuda()
for emu in (8, 0):
    _native.context().set("emu_slices", emu)
    g = solver.BuildGraph(inp, nrhs=8)
    print("emu", emu, list(zip([n for n, _ in g.stages], g.stage_launches)), flush=True)
    g.load(inp, F)
    st = g.replay_build(); U = g.replay_solve(); torch.cuda.synchronize()
    st2 = solver.build_device(inp); U2 = solver.solve_device(st2, F); torch.cuda.synchronize()
    print("graph vs eager root T equal:", torch.equal(st.root_T.device_tensor, st2.root_T.device_tensor), "U equal:", torch.equal(U, U2), flush=True)
