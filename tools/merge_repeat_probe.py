"""Re-run one merge level on fixed child T and diff the workspace pieces across runs (dev tool)."""
import sys, ctypes
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems, _native
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dtarget = int(sys.argv[2]) if len(sys.argv) > 2 else 10
c = problems.CONFIGS[cfg]
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
inp = solver.prepare(tree, nodes, c.coefficients())
st = solver.build_device(inp, keep_level_T=True)
torch.cuda.synchronize()
lib = _native.load()
lay, dl = inp.layout, inp.dev_layout
dlay = lay.depths[dtarget]
nb, n3, ne, m = dlay.n_boxes, dlay.n3, dlay.ne, dlay.m
child = st.level_T[dtarget + 1]
print("ngroups", inp.ngroups, "nb", nb, "n3", n3, "ne", ne)
outs = []
for r in range(4):
    S = torch.empty((nb, n3, ne), dtype=torch.float64, device="cuda")
    T = torch.empty((nb, ne, ne), dtype=torch.float64, device="cuda")
    wsb = lib.hps_merge_workspace_bytes(nb, n3, ne)
    ws = torch.full((wsb // 8,), float(r), dtype=torch.float64, device="cuda")  # different garbage per run
    status = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    _native.check(lib.hps_merge_level(_native.context(), nb, n3, ne, m, lay.q, _native.ptr(child), ne_c := child.shape[-1] ** 2 if False else child.shape[1] * child.shape[2],
                                      None, _native.ptr(dl.maps[dtarget]), _native.ptr(dl.vmode[dtarget]),
                                      _native.ptr(S), _native.ptr(T), _native.ptr(ws), wsb,
                                      ctypes.c_void_p(status.data_ptr()), 0, _native.stream_ptr()), "merge")
    torch.cuda.synchronize()
    X = ws[: nb * n3 * n3].view(nb, n3, n3).clone()
    R = ws[nb * n3 * n3: nb * n3 * (n3 + ne)].clone()
    Cm = ws[nb * n3 * (n3 + ne): nb * n3 * (n3 + 2 * ne)].clone()
    outs.append((X, R, Cm, S, T))
for r in range(1, 4):
    names = ["Xinv", "R", "C", "S", "T"]
    res = []
    for nm, a, b in zip(names, outs[0], outs[r]):
        neq = (a != b)
        if neq.dim() == 3:
            bad = torch.nonzero(neq.flatten(1).any(1)).flatten().tolist()
        else:
            bad = [int(neq.sum())]
        res.append(f"{nm}: eq={bool(not neq.any())} bad={bad[:8]}")
    print(f"run {r}:", "; ".join(res))
