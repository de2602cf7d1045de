"""Parity of the CUDA path (through the C ABI) against the reference's golden vectors and the
oracle, on null-mode-invariant quantities. Run on a B200: pytest -m gpu.

Gates (relative, max|diff| / max|ref|): leaf T / Psi <= 1e-12, merged/root T <= 1e-10
(1e-8 for the Helmholtz configs 3, 4), per-leaf Chebyshev boundary values L1 u <= 1e-10
(1e-8 Helmholtz). Tree/index layout is bit-exact (tests/test_layout.py)."""
import numpy as np
import pytest
import torch

import paper_1307_2665_b200 as P
from oracle import hps_oracle as O
from paper_1307_2665_b200 import instrumentation, problems, solver

from _util import coeff_dict, golden, rel

pytestmark = pytest.mark.gpu
T_TOL = {1: 1e-10, 2: 1e-10, 3: 1e-8, 4: 1e-8, 5: 1e-10}
U_TOL = T_TOL


def gpu_build(cfg, L, **kw):
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
    st = solver.build(tree, nodes, problems.coefficients(cfg), switch_threshold=None, **kw)
    return tree, nodes, st


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_against_reference_golden_L2(cfg):
    g = golden(f"cfg{cfg}_L2.npz")
    tree, nodes, st = gpu_build(cfg, 2, keep_level_T=True)
    k = g["leaf_T"].shape[0]
    assert rel(st.T_leaf_groups.cpu().numpy()[:k], g["leaf_T"]) < 1e-12
    assert rel(st.psi_groups.cpu().numpy()[:g["psi"].shape[0]], g["psi"]) < 1e-12
    assert rel(st._cond.cpu().numpy(), g["cond"]) < 1e-12
    assert np.array_equal(st.leaf_group, g["leaf_group"])
    lt = st.level_T[3].cpu().numpy()  # leaf-pair depth 2L-1 = 3: boxes 7, 8 are slots 0, 1
    for slot, box in ((0, 7), (1, 8)):
        assert rel(lt[slot], g[f"T_box{box}"]) < T_TOL[cfg]
        assert rel(st.S[box].dense, g[f"S_box{box}"]) < T_TOL[cfg]  # X nonsingular at this depth
    assert rel(st.root_T.dense, g["root_T"]) < T_TOL[cfg]
    u = solver.solve(st, g["F"])
    ot = O.build_tree((0, 1, 0, 1), 2, 16)
    L1u = np.stack([st.geometry.L1 @ u[ot.I_e[b]] for b in ot.leaves])
    assert rel(L1u, g["L1u"]) < U_TOL[cfg]


@pytest.mark.parametrize("cfg,L", [(1, 3), (2, 3), (2, 4), (3, 3), (4, 4), (5, 4), (1, 5)])
def test_every_operator_against_oracle(cfg, L):
    tree, nodes, st = gpu_build(cfg, L, keep_level_T=True)
    ot = O.build_tree((0, 1, 0, 1), L, 16)
    ost = O.build(ot, coeff_dict(problems.coefficients(cfg)), keep_T=True)
    assert rel(st.T_leaf_groups.cpu().numpy(), ost.T_groups) < 1e-12
    assert rel(st.psi_groups.cpu().numpy(), ost.psi_groups) < 1e-12
    assert rel(st._cond.cpu().numpy(), ost.cond) < 1e-12
    worst = 0.0
    for d in range(2 * L):
        Td = st.level_T[d].cpu().numpy()
        for k in range(Td.shape[0]):
            worst = max(worst, rel(Td[k], ost.T[(1 << d) - 1 + k]))
    assert worst < T_TOL[cfg], worst
    F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=7, batch=3)
    u = solver.solve(st, F)
    uo = O.solve(ost, F)
    assert rel(O.leaf_cheb_boundary(ost, u), O.leaf_cheb_boundary(ost, uo)) < U_TOL[cfg]
    assert rel(O.leaf_flux(ost, u), O.leaf_flux(ost, uo)) < U_TOL[cfg]
    assert rel(O.leaf_cheb_field(ost, u), O.leaf_cheb_field(ost, uo)) < U_TOL[cfg]


@pytest.mark.parametrize("cfg,L,tol", [(1, 3, 1e-11), (1, 6, 1e-9), (3, 4, 1e-7), (3, 7, 1e-9)])
def test_exact_solution(cfg, L, tol):
    """cfg 1: exp(x1) sin(x2); cfg 3: plane wave, also at its BASELINE size (L = 7, 4.2e6 unknowns;
    measured 6e-11). Checked on the invariant L1 u."""
    tree, nodes, st = gpu_build(cfg, L)
    F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=4, batch=1)
    u = solver.solve(st, F)
    ex = problems.exact_solution(cfg, nodes.points[:, 0], nodes.points[:, 1], seed=4, batch=1)
    lay = st.layout
    L1 = st.geometry.L1
    got = np.einsum("rc,lc->lr", L1, u[lay.leaf_I_e])
    want = np.einsum("rc,lc->lr", L1, ex[lay.leaf_I_e])
    assert rel(got, want) < tol


def test_full_size_cfg2_against_oracle():
    """BASELINE config 2 at its full size (L=6, 4096 leaf groups): root DtN + invariants."""
    cfg, L = 2, 6
    tree, nodes, st = gpu_build(cfg, L)
    ot = O.build_tree((0, 1, 0, 1), L, 16)
    ost = O.build(ot, coeff_dict(problems.coefficients(cfg)))
    assert rel(st.root_T.dense, ost.root_T) < 1e-10
    F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0, batch=4)
    u = solver.solve(st, F)
    assert rel(O.leaf_cheb_boundary(ost, u), O.leaf_cheb_boundary(ost, O.solve(ost, F))) < 1e-10


@pytest.mark.parametrize("cfg,L", [(1, 6), (2, 6), (5, 7), (5, 9), (4, 8)])
def test_full_size_properties(cfg, L):
    """Size-independent properties at BASELINE sizes (config 5 at L = 9: 6.7e7 unknowns, 8.6 GB
    root DtN): constants are in the DtN null space for operators with no
    zeroth-order term, and the solve is linear."""
    tree, nodes, st = gpu_build(cfg, L)
    T = st.root_T.device_tensor
    one = torch.ones(T.shape[0], dtype=torch.float64, device=T.device)
    if cfg != 4:  # config 4 (variable Helmholtz) has a zeroth-order term: linearity only
        assert float((T @ one).abs().max() / T.abs().max()) < 1e-10
    F = problems.boundary_data(2, nodes.points[tree.root.I_e], seed=9, batch=2)
    u = solver.solve(st, F)
    uc = solver.solve(st, 2.0 * F[:, 0] - 3.0 * F[:, 1])
    L1 = st.geometry.L1
    Ie = st.layout.leaf_I_e
    lin = np.einsum("rc,lc->lr", L1, 2.0 * u[Ie, 0] - 3.0 * u[Ie, 1])
    assert rel(np.einsum("rc,lc->lr", L1, uc[Ie]), lin) < 1e-11


def test_laplace_dtn_on_linear_data():
    """Leaf/root T on u = x1: flux 1 on vertical edges, 0 on horizontal."""
    tree, nodes, st = gpu_build(1, 3)
    ids = tree.root.I_e
    x = nodes.points[ids, 0]
    v = solver.apply_global_dtn(st, x)
    vert = nodes.on_vertical[ids]
    assert np.abs(v[vert] - 1.0).max() < 1e-9 and np.abs(v[~vert]).max() < 1e-9
    Tl = st.T_leaf_groups[0].cpu().numpy()
    leaf = tree.boxes[tree.n_boxes - 1]
    xl = nodes.points[leaf.I_e, 0]
    fl = Tl @ xl
    assert np.abs(fl[16:32] - 1).max() < 1e-10 and np.abs(fl[:16]).max() < 1e-10
    assert np.abs(Tl @ np.ones(64)).max() < 1e-9 * np.abs(Tl).max()


def test_repeat_solve_and_build_are_bitwise_deterministic():
    tree, nodes, st = gpu_build(2, 4)
    F = problems.boundary_data(2, nodes.points[tree.root.I_e], seed=1, batch=16)
    u1 = solver.solve(st, F)
    u2 = solver.solve(st, F)
    assert np.array_equal(u1, u2)
    _, _, st2 = gpu_build(2, 4)
    assert torch.equal(st.root_T.device_tensor, st2.root_T.device_tensor)
    assert all(torch.equal(a, b) for a, b in zip(st.S_levels, st2.S_levels))


def test_full_size_constant_coefficient_build_is_bitwise_deterministic():
    # cfg3 at full size exposed a cross-CTA race on max|diag X| in the deflation (fixed r01): every
    # build of the same input must give bit-identical S and T at every depth.
    c = problems.CONFIGS[3]
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), c.L, 16)
    inp = solver.prepare(tree, nodes, c.coefficients())
    ref = solver.build_device(inp, keep_level_T=True)
    for _ in range(3):
        st = solver.build_device(inp, keep_level_T=True)
        for d in range(len(ref.S_levels)):
            assert torch.equal(ref.S_levels[d], st.S_levels[d]), f"S differs at depth {d}"
            assert torch.equal(ref.level_T[d], st.level_T[d]), f"T differs at depth {d}"
        del st


def test_batched_solve_matches_single_rhs():
    tree, nodes, st = gpu_build(2, 3)
    F = problems.boundary_data(2, nodes.points[tree.root.I_e], seed=2, batch=20)
    U = solver.solve(st, F)  # GEMM path (b > 8)
    U4 = solver.solve(st, F[:, :4])  # warp-per-row path
    for j in (0, 7, 19):
        uj = solver.solve(st, F[:, j])
        assert rel(U[:, j], uj) < 1e-13
    assert rel(U4, U[:, :4]) < 1e-13


def test_counters_and_stage_separation():
    instrumentation.counts.clear()
    tree, nodes, st = gpu_build(2, 2)
    snap = instrumentation.snapshot()
    assert snap["merge"] == 15 and snap["leaf_dtn"] == 1
    solver.solve(st, lambda x, y: x * y)
    after = instrumentation.snapshot()
    assert after["solve"] == 1 and after["merge"] == 15 and after["leaf_dtn"] == 1
    solver.apply_global_dtn(st, lambda x, y: x)
    assert instrumentation.snapshot()["apply_dtn"] == 1
    with pytest.raises(ValueError):
        solver.solve(st, np.zeros(5))


def _owner(tree, x, y):
    # the reference's owning-leaf rule (solver.py:330-346), restated for the tests
    n, dom = 1 << tree.levels, tree.domain

    def cell(t, extent):
        s = (t / extent) * n
        i = int(np.floor(s))
        if i == s and i > 0:
            i -= 1
        return min(max(i, 0), n - 1)

    return tree.leaf_at(cell(x - dom.x_lo, dom.width), cell(y - dom.y_lo, dom.height))


def _oracle_point_values(tree, st, W, pts, deriv=False):
    # rx W ry^T (or the boundary-flux derivative) from oracle leaf fields W (n_leaf, p*p[, b])
    dom, g = tree.domain, st.geometry
    out = []
    for (x, y) in pts:
        leaf = _owner(tree, x, y)
        Wk = W[leaf.index - (4 ** tree.levels - 1)]
        Wk = Wk.reshape((16, 16) + Wk.shape[1:])
        rx = P.grid.interp_matrix(g.cheb_x, [x - leaf.rect.x_lo])[0]
        ry = P.grid.interp_matrix(g.cheb_y, [y - leaf.rect.y_lo])[0]
        if deriv:
            on_v, on_h = x in (dom.x_lo, dom.x_hi), y in (dom.y_lo, dom.y_hi)
            if on_v and not on_h:
                rx = rx @ g.Dx
            else:
                ry = ry @ g.Dy
        out.append(np.einsum("i,ij...,j->...", rx, Wk, ry))
    return np.array(out)


def test_state_api_against_oracle():
    cfg, L = 2, 2
    tree, nodes, st = gpu_build(cfg, L)
    ot = O.build_tree((0, 1, 0, 1), L, 16)
    ost = O.build(ot, coeff_dict(problems.coefficients(cfg)))
    f = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=3, batch=1)
    assert rel(solver.apply_global_dtn(st, f), ost.root_T @ f) < 1e-12
    u = solver.solve(st, f)
    pts = [(0.13, 0.71), (0.5, 0.5), (0.999, 0.0001), (0.25, 0.75)]
    uo = O.solve(ost, f)
    # post_process is null-mode invariant: compare against the oracle-state evaluation
    W = O.leaf_cheb_field(ost, uo)
    ref = []
    for (x, y) in pts:
        leaf = _owner(tree, x, y)
        k = leaf.index - (4 ** L - 1)
        Wk = W[k].reshape(16, 16)
        rx = P.grid.interp_matrix(st.geometry.cheb_x, [x - leaf.rect.x_lo])
        ry = P.grid.interp_matrix(st.geometry.cheb_y, [y - leaf.rect.y_lo])
        ref.append(float((rx @ Wk @ ry.T)[0, 0]))
    assert rel(solver.post_process(st, u, pts), np.array(ref)) < 1e-10
    bpts = [(0.0, 0.3), (1.0, 0.6), (0.2, 0.0), (0.7, 1.0)]
    assert np.all(np.isfinite(solver.boundary_flux_at(st, u, bpts)))
    rep = solver.memory_report(st)
    ni, nb = 196, 60
    S_entries = sum(ost.S[b].size for b in ost.S)
    want = ost.root_T.size + st.n_leaf_groups * ni * nb + st.geometry.L1.size + st.geometry.L4.size + S_entries
    assert rep["total_entries"] == want
    assert st.S[0].dense.shape == ost.S[0].shape and len(st.psi) == 16


def test_distributed_path_single_rank_cuda_backend():
    """parallel.py with the CUDA backend at world size 1 (the exchange itself is covered by the
    gloo tests in test_distributed.py) equals the single-process build."""
    import os
    import socket

    import torch.distributed as dist

    from paper_1307_2665_b200 import parallel

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        tree, nodes, st = gpu_build(2, 3)
        be = parallel.CudaBackend(tree)
        comm = parallel.TorchComm()
        ds = parallel.build_distributed(tree, problems.coefficients(2), comm, be)
        assert rel(ds.root_T[0].cpu().numpy(), st.root_T.dense) < 1e-13
        F = torch.from_numpy(problems.boundary_data(2, nodes.points[tree.root.I_e], seed=2, batch=5)).cuda()
        u = parallel.solve_distributed(ds, F, comm)
        full = parallel.gather_solution(ds, u, comm, 5)
        assert rel(full, solver.solve(st, F.cpu().numpy())) < 1e-13
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q,L,cfg", [(21, 2, 2), (12, 3, 1), (10, 2, 3), (7, 3, 5), (21, 4, 2), (12, 5, 2)])
def test_general_q_against_oracle(q, L, cfg):
    """Any q >= 3 (the paper uses q = 21): generic leaf kernel, unaligned GEMM path, unequal
    recursive-inverse halves; at (21, 4) and (12, 5) the look-ahead interface inverse runs too
    (parent interfaces of 168..336 and 192..384 nodes)."""
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, q)
    st = solver.build(tree, nodes, problems.coefficients(cfg), keep_level_T=True)
    ot = O.build_tree((0, 1, 0, 1), L, q)
    ost = O.build(ot, coeff_dict(problems.coefficients(cfg)), keep_T=True)
    assert rel(st.T_leaf_groups.cpu().numpy(), ost.T_groups) < 1e-12
    assert rel(st.root_T.dense, ost.root_T) < T_TOL[cfg]
    F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=1, batch=12)
    u = solver.solve(st, F)
    assert rel(O.leaf_cheb_boundary(ost, u), O.leaf_cheb_boundary(ost, O.solve(ost, F))) < U_TOL[cfg]


@pytest.mark.parametrize("n,batch", [(16, 7), (100, 3), (128, 2), (168, 2), (336, 1), (512, 2)])
def test_inverse_batched(n, batch):
    from paper_1307_2665_b200 import _native

    lib = _native.load()
    rng = np.random.default_rng(n)
    A = rng.standard_normal((batch, n, n)) + 3 * np.sqrt(n) * np.eye(n)
    X = torch.from_numpy(A.copy()).cuda()
    ws = torch.empty(lib.hps_inverse_workspace_bytes(n, batch), dtype=torch.uint8, device="cuda")
    stw = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    _native.check(lib.hps_inverse_batched(_native.context(), n, batch, _native.ptr(X), n, n * n, _native.ptr(ws), ws.numel(),
                                          _native.ptr(stw), _native.stream_ptr()), "inverse")
    Xi = X.cpu().numpy()
    assert np.abs(A @ Xi - np.eye(n)).max() < 1e-11
    assert int(stw.item()) == -1


def test_pipeline_matches_sequential_build_and_solve():
    # solver.Pipeline overlaps the host preparation of job i+1 with the device work of job i; every
    # job's u must be bitwise equal to a plain build + solve of that job alone.
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 4, 16)
    pts = nodes.points[tree.root.I_e]
    jobs = [(problems.coefficients(cfg), problems.boundary_data(2, pts, seed=cfg, batch=3)) for cfg in (2, 4, 3, 2)]
    # streams>1: consecutive jobs on alternating compute streams, split-K scratch in separate slots
    for graphs, streams in ((False, 1), (True, 1), (False, 2), (True, 2), (True, 3)):
        pipe = solver.Pipeline(tree, nodes, reuse_graphs=graphs, streams=streams)
        got = [(U[:, :3].numpy().copy(), st.n_leaf_groups) for U, st in pipe.run(jobs)]
        got += [(U[:, :3].numpy().copy(), st.n_leaf_groups) for U, st in pipe.run(jobs)]  # counters carry over
        pipe.close()
        assert len(got) == 2 * len(jobs)
        for (co, F), (u, ng) in zip(jobs + jobs, got):
            st = solver.build(tree, nodes, co)
            assert ng == st.n_leaf_groups
            assert np.array_equal(u, solver.solve(st, F))


@pytest.mark.parametrize("cfg,L", [(2, 2), (4, 3)])
def test_device_post_processing_against_oracle_fields(cfg, L):
    # hps_leaf_fields / hps_eval_points vs the oracle's null-mode-invariant leaf fields
    tree, nodes, st = gpu_build(cfg, L)
    ot = O.build_tree((0, 1, 0, 1), L, 16)
    ost = O.build(ot, coeff_dict(problems.coefficients(cfg)))
    F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=5, batch=3)
    U = solver.solve(st, F)
    Wo = O.leaf_cheb_field(ost, O.solve(ost, F))          # (n_leaf, p*p, 3)
    tol = 1e-10 if cfg in (1, 2, 5) else 1e-8
    Wd = solver.leaf_fields(st, U).cpu().numpy()          # (n_leaf, p, p, 3)
    assert rel(Wd.reshape(Wo.shape), Wo) < tol
    w1 = solver.leaf_fields(st, U[:, 1]).cpu().numpy()    # vector input
    assert rel(w1.reshape(Wo.shape[:2]), Wo[:, :, 1]) < tol
    rng = np.random.default_rng(7)
    pts = np.concatenate([rng.uniform(0, 1, (50, 2)), [[0.5, 0.5], [0.25, 0.75], [0.0, 0.0], [1.0, 1.0], [0.125, 1.0]]])
    got = solver.post_process(st, U, pts)
    assert got.shape == (len(pts), 3)
    assert rel(got, _oracle_point_values(tree, st, Wo, pts)) < tol
    assert rel(solver.post_process(st, U[:, 0], pts), got[:, 0]) < 1e-14
    bpts = [(0.0, 0.3), (1.0, 0.6), (0.2, 0.0), (0.7, 1.0), (0.0, 0.0), (1.0, 0.5)]
    assert rel(solver.boundary_flux_at(st, U, bpts), _oracle_point_values(tree, st, Wo, bpts, deriv=True)) < tol
    with pytest.raises(ValueError):
        solver.post_process(st, U, [(1.5, 0.5)])
    with pytest.raises(ValueError):
        solver.boundary_flux_at(st, U, [(0.5, 0.5)])


def test_gauge_fixed_solution_laplace_exact_and_invariant():
    # Gauss-node u re-tabulated from the leaf fields: physical (matches the exact solution),
    # keeps the Dirichlet data on the outer boundary, and equals the oracle re-tabulation
    cfg, L = 1, 3
    tree, nodes, st = gpu_build(cfg, L)
    f = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0)
    u = solver.solve(st, f)
    ug = solver.gauge_fixed_solution(st, u).cpu().numpy()
    ex = problems.exact_solution(cfg, nodes.points[:, 0], nodes.points[:, 1])
    assert np.max(np.abs(ug - ex)) < 1e-10
    root_ie = np.asarray(tree.root.I_e)
    assert np.array_equal(ug[root_ie], np.asarray(f, dtype=float))
    # oracle re-tabulation: per leaf sides Qx W[:,0], Qy W[p-1,:], Qx W[:,p-1], Qy W[0,:], averaged
    ot = O.build_tree((0, 1, 0, 1), L, 16)
    ost = O.build(ot, coeff_dict(problems.coefficients(cfg)))
    Wo = O.leaf_cheb_field(ost, O.solve(ost, f)).reshape(-1, 16, 16)
    g = st.geometry
    acc, cnt = np.zeros(nodes.N), np.zeros(nodes.N)
    for k, b in enumerate(ot.leaves):
        Wk = Wo[k]
        side = np.concatenate([g.Qx @ Wk[:, 0], g.Qy @ Wk[15, :], g.Qx @ Wk[:, 15], g.Qy @ Wk[0, :]])
        np.add.at(acc, ot.I_e[b], side)
        np.add.at(cnt, ot.I_e[b], 1.0)
    ref = acc / cnt
    ref[root_ie] = f
    assert rel(ug, ref) < 1e-12
    ug2 = solver.gauge_fixed_solution(st, u).cpu().numpy()
    assert np.array_equal(ug, ug2)


def test_build_graph_replays_equal_eager_builds():
    # solver.BuildGraph: a captured build + batched solve replayed with new inputs must give the
    # same bits as an eager build and solve of those inputs
    from paper_1307_2665_b200.leafops import CoefficientField
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 4, 16)
    pts = nodes.points[tree.root.I_e]
    co = [CoefficientField(c11=lambda x, y, a=a: 1.0 + a * np.sin(3 * x) * np.cos(2 * y), c22=lambda x, y: 1.0 + 0.3 * x * y)
          for a in (0.1, 0.4, 0.25)]
    F = [problems.boundary_data(2, pts, seed=s, batch=5) for s in range(3)]
    inps = [solver.prepare(tree, nodes, c) for c in co]
    g = solver.BuildGraph(inps[0], nrhs=5)
    assert g.launches > 0
    for inp, Fk, c in zip(inps, F, co):
        st, U = g.run(inp, Fk)
        solver.check_build(st)
        got_T = st.root_T.device_tensor.clone()
        got_U = U[:, :5].clone()
        ref = solver.build_device(inp)
        Uref = solver.solve_device(ref, torch.from_numpy(np.ascontiguousarray(Fk)).cuda())
        assert torch.equal(got_T, ref.root_T.device_tensor)
        assert torch.equal(got_U, Uref[:, :5])
        assert rel(solver.post_process(st, U[:, :5], [(0.3, 0.6)]), solver.post_process(ref, Uref[:, :5], [(0.3, 0.6)])) == 0
