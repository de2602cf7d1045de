"""The pivoted LU behind the large interface systems (n3 > 128), through the C ABI (GPU only).

Reference: merge.py:106-110 (scipy.linalg.lu_factor / lu_solve, LAPACK getrf / getrs, partial
pivoting over the whole column). The device LU must pick the same pivot rows as LAPACK on generic
matrices, solve to working accuracy, and survive matrices whose leading blocks are singular (where a
factorisation pivoting only inside 128-blocks breaks down)."""
import numpy as np
import pytest
import scipy.linalg as sla
import torch

from paper_1307_2665_b200 import _native

from _util import rel

pytestmark = pytest.mark.gpu


def lu_solve_gpu(A, R):
    lib = _native.load()
    batch, n, _ = A.shape
    ne = R.shape[2]
    X = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    Rt = torch.from_numpy(np.ascontiguousarray(R)).cuda()
    S = torch.empty((batch, n, ne), dtype=torch.float64, device="cuda")
    piv = torch.empty((batch, n), dtype=torch.int32, device="cuda")
    wsb = lib.hps_lu_workspace_bytes(n, batch)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    stw = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    _native.check(lib.hps_lu_solve_batched(_native.context(), n, ne, batch, _native.ptr(X), _native.ptr(Rt),
                                           _native.ptr(S), _native.ptr(piv), _native.ptr(ws), wsb, _native.ptr(stw),
                                           _native.stream_ptr()), "lu")
    return X.cpu().numpy(), S.cpu().numpy(), piv.cpu().numpy(), int(stw.item())


@pytest.mark.parametrize("n,ne,batch", [(144, 64, 3), (256, 96, 2), (400, 130, 1), (1024, 256, 2), (2048, 64, 1),
                                        (4096, 32, 1)])
def test_lu_matches_lapack(n, ne, batch):
    """Same pivots as LAPACK getrf, same L\\U, S = X^-1 R to working accuracy; 2048 and 4096 rows run the
    panel as a 2- and 4-CTA cluster."""
    rng = np.random.default_rng(n + ne)
    A = rng.standard_normal((batch, n, n))
    R = rng.standard_normal((batch, n, ne))
    LU, S, piv, st = lu_solve_gpu(A, R)
    assert st == -1
    for b in range(batch):
        lu_ref, piv_ref = sla.lu_factor(A[b])
        agree = np.mean(piv[b] == piv_ref)
        assert agree >= 0.999, agree  # near-ties (within rounding) may legitimately differ
        if agree == 1.0:
            assert rel(LU[b], lu_ref) < 1e-10
        want = np.linalg.solve(A[b], R[b])
        resid = np.abs(A[b] @ S[b] - R[b]).max() / (np.abs(A[b]).max() * np.abs(S[b]).max() * n)
        assert resid < 1e-15, resid
        assert rel(S[b], want) < 1e-9 * np.linalg.cond(A[b]) / n


def test_lu_pivots_across_blocks():
    """X = [[0, B], [C, D]]: every leading 128-block is singular, X is well conditioned. Pivoting inside
    the 128-blocks only (the recursive block inverse) cannot factor it; the full-column LU does."""
    rng = np.random.default_rng(5)
    n, ne, h = 512, 48, 256
    B = rng.standard_normal((h, h)) + 4 * np.sqrt(h) * np.eye(h)
    C = rng.standard_normal((h, h)) + 4 * np.sqrt(h) * np.eye(h)
    X = np.zeros((n, n))
    X[:h, h:] = B
    X[h:, :h] = C
    X[h:, h:] = rng.standard_normal((h, h))
    R = rng.standard_normal((1, n, ne))
    _, S, piv, st = lu_solve_gpu(X[None], R)
    assert st == -1
    assert rel(S[0], np.linalg.solve(X, R[0])) < 1e-12
    assert np.array_equal(piv[0], sla.lu_factor(X)[1])


def test_lu_flags_singular_matrix():
    rng = np.random.default_rng(9)
    n = 256
    A = rng.standard_normal((2, n, n))
    A[1, :, 7] = 0.0  # exactly singular second matrix
    _, S, _, st = lu_solve_gpu(A, rng.standard_normal((2, n, 16)))
    assert st == 1
    assert np.isfinite(S[0]).all()


def _big_depths(lay):
    return {d for d in range(len(lay.depths)) if lay.depths[d].n3 > 128}


@pytest.mark.parametrize("cfg,L", [(2, 5), (4, 5), (5, 6)])
def test_pivoted_build_matches_fast_build(cfg, L):
    """The whole build with every interface of n3 > 128 on the pivoted LU agrees with the default
    (residual-checked block inverse) build: root DtN and the invariant solution."""
    import paper_1307_2665_b200 as P
    from paper_1307_2665_b200 import problems, solver
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
    inp = solver.prepare(tree, nodes, problems.coefficients(cfg))
    fast = solver.build_device(inp)
    assert solver.check_build(fast) == set()
    piv = solver.build_device(inp, pivoted=_big_depths(inp.layout))
    assert solver.check_build(piv) == set()
    tol = 1e-8 if cfg == 4 else 1e-11
    assert rel(piv.root_T.dense, fast.root_T.dense) < tol
    F = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=2, batch=3)
    Ie = inp.layout.leaf_I_e
    L1 = fast.geometry.L1
    a = np.einsum("rc,lcb->lrb", L1, solver.solve(fast, F)[Ie])
    b = np.einsum("rc,lcb->lrb", L1, solver.solve(piv, F)[Ie])
    assert rel(b, a) < tol * 10


def test_failed_residual_check_falls_back_to_pivoted_lu():
    """An interface whose leading 128-block is singular (the block inverse pivots only inside
    128-blocks): the fast path's residual check raises the status word to HPS_STATUS_PIVOT + merge;
    the pivoted path (HPS_MERGE_PIVOTED) then solves it, and T = blkdiag + C S matches numpy."""
    import paper_1307_2665_b200 as P
    from paper_1307_2665_b200 import solver
    from paper_1307_2665_b200.grid import layout_of

    lib = _native.load()
    tree, _ = P.build_tree(P.Rectangle(0, 1, 0, 1), 4, 16)
    lay = layout_of(tree)
    geom = P.LeafGeometry.get(16, tree.leaf_width, tree.leaf_height)
    dl_dev = solver._DeviceLayout.get(lay, geom, torch.device("cuda"))
    d = 0
    dl = lay.depths[d]
    n3, ne, m, q = dl.n3, dl.ne, dl.m, 16
    rng = np.random.default_rng(0)
    Ta = rng.standard_normal((m, m))
    Tb = rng.standard_normal((m, m))
    # X = Ta[j3a, j3a] - Tb[j3b, j3b] with an exactly zero leading 128 x 128 block, plus a strong
    # off-diagonal coupling so the whole X is well conditioned
    Xw = rng.standard_normal((n3, n3))
    h = 128
    Xw[:h, :h] = 0.0
    Xw[:h, h:] += 8 * np.sqrt(n3) * np.eye(h, n3 - h)
    Xw[h:, :h] += 8 * np.sqrt(n3) * np.eye(n3 - h, h)
    Ta[np.ix_(dl.j3a, dl.j3a)] = Xw + Tb[np.ix_(dl.j3b, dl.j3b)]
    kids = torch.from_numpy(np.stack([Ta, Tb])).cuda()
    outs = {}
    for flags in (0, _native.HPS_MERGE_PIVOTED):
        S = torch.empty((1, n3, ne), dtype=torch.float64, device="cuda")
        T = torch.empty((1, ne, ne), dtype=torch.float64, device="cuda")
        wsb = lib.hps_merge_workspace_bytes(1, n3, ne)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        stw = torch.full((1,), -1, dtype=torch.int32, device="cuda")
        _native.check(lib.hps_merge_level_ahead(
            _native.context(), 1, n3, ne, m, q, _native.ptr(kids), m * m, None, _native.ptr(dl_dev.maps[d]),
            _native.ptr(dl_dev.vmode[d]), _native.ptr(S), _native.ptr(T), _native.ptr(ws), wsb, _native.ptr(stw), 0, 0,
            None, 0, 0, None, None, 0, None, 0, flags, _native.stream_ptr()), "merge")
        outs[flags] = (int(stw.item()), S.cpu().numpy()[0], T.cpu().numpy()[0])
    assert outs[0][0] >= _native.HPS_STATUS_PIVOT  # the check caught the breakdown
    st, S, T = outs[_native.HPS_MERGE_PIVOTED]
    assert st == -1
    X = Ta[np.ix_(dl.j3a, dl.j3a)] - Tb[np.ix_(dl.j3b, dl.j3b)]
    R = np.concatenate([-Ta[np.ix_(dl.j3a, dl.j1a)], Tb[np.ix_(dl.j3b, dl.j2b)]], axis=1)
    C = np.concatenate([Ta[np.ix_(dl.j1a, dl.j3a)], Tb[np.ix_(dl.j2b, dl.j3b)]])
    n1 = ne // 2
    blk = np.zeros((ne, ne))
    blk[:n1, :n1] = Ta[np.ix_(dl.j1a, dl.j1a)]
    blk[n1:, n1:] = Tb[np.ix_(dl.j2b, dl.j2b)]
    # the deflated system's solution satisfies X S = R up to the corner-mode components, which C annihilates
    # only for genuine DtN maps; here check the solve itself against the deflated matrix
    vm = dl_dev.vmode[d].cpu().numpy()
    vs, ve = vm[:q], vm[q:]
    V = np.zeros((n3, n3 // q - 1))
    for k in range(n3 // q - 1):
        V[k * q:(k + 1) * q, k] = ve
        V[(k + 1) * q:(k + 2) * q, k] = vs
    Xd = X + np.abs(np.diag(X)).max() * V @ V.T
    Sw = np.linalg.solve(Xd, R)
    assert rel(S, Sw) < 1e-10
    assert rel(T, blk + C @ Sw) < 1e-10
