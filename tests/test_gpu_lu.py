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
