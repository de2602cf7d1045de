"""Fake multi-GPU: the 2/4/8-way subtree partition run as threads on ONE device, device-to-device
copies in place of NCCL (parallel.LocalComm). Per-box arithmetic is the same
as the single-process build, so the results must agree BITWISE: every S, the root DtN map and the
solution. Split-K is off in every context (it is the only batch-dependent summation order) and the
look-ahead inverse is off (it forms X along a different arithmetic path); nothing else changes.
Reference sweep: solver.py:266-285 (build), 303-316 (solve)."""
import numpy as np
import pytest
import torch

import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import _native, parallel, problems, solver

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,cfg,L,mode", [(2, 2, 4, "panels"), (4, 3, 4, "panels"), (8, 2, 4, "panels"),
                                              (4, 4, 4, "owner"), (8, 5, 5, "panels")])
def test_partitioned_build_and_solve_are_bitwise_equal(world, cfg, L, mode, monkeypatch):
    monkeypatch.setenv("HPS_AHEAD_MIN_N3", "0")
    ctxs = [_native.context(slot) for slot in range(world + 1)]
    for c in ctxs:
        c.set("splitk", 0)
    try:
        tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
        co = problems.coefficients(cfg)
        st1 = solver.build(tree, nodes, co)
        F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=3, batch=5)
        u1 = solver.solve(st1, F)

        def rank_fn(comm):
            be = parallel.CudaBackend(tree, ctx_slot=comm.rank + 1)
            st = parallel.build_distributed(tree, co, comm, be, top_mode=mode)
            Ft = torch.from_numpy(np.ascontiguousarray(F)).cuda() if comm.rank == 0 else None
            u = parallel.solve_distributed(st, Ft, comm)
            full = parallel.gather_solution(st, u, comm, F.shape[1])
            torch.cuda.synchronize()
            return st, full

        res = parallel.LocalComm.run(world, rank_fn)
        st0, full = res[0]
        assert torch.equal(st0.root_T[0], st1.root_T.device_tensor)
        n_s = 0
        for r, (st, _) in enumerate(res):
            for d, S in st.S_local.items():
                lo, hi = st.plan.local_slots(r, d)
                assert torch.equal(S, st1.S_levels[d][lo:hi]), (r, d)
                n_s += hi - lo
            for d, S in st.S_top.items():
                k = st.plan.top_boxes(r, d)[0]
                assert torch.equal(S[0], st1.S_levels[d][k]), (r, d)
                n_s += 1
        assert n_s == (1 << (2 * L)) - 1  # every parent box exactly once
        assert np.array_equal(full, u1)
    finally:
        for c in ctxs:
            c.set("splitk", 1)
