"""Unit tests of the CUDA kernels through the C ABI (GPU only)."""
import numpy as np
import pytest
import torch

from paper_1307_2665_b200 import _native

from _util import rel

pytestmark = pytest.mark.gpu


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("M,N,K,B,alpha,beta", [(64, 64, 16, 1, 1.0, 0.0), (96, 96, 16, 3, -1.0, 1.0),
                                                (256, 512, 128, 2, 0.5, 2.0), (1000, 130, 64, 1, 1.0, 0.0),
                                                (128, 128, 32, 300, 1.0, 1.0), (16, 8, 16, 7, 2.0, 0.0),
                                                (1024, 1024, 512, 1, 1.0, -1.0)])
def test_dgemm(M, N, K, B, alpha, beta):
    lib = _native.load()
    rng = np.random.default_rng(M + N + K)
    A, Bm, C = rng.standard_normal((B, M, K)), rng.standard_normal((B, K, N)), rng.standard_normal((B, M, N))
    tA, tB, tC = cuda(A), cuda(Bm), cuda(C)
    _native.check(lib.hps_dgemm_batched(_native.context(), M, N, K, B, alpha, _native.ptr(tA), K, M * K, _native.ptr(tB), N, K * N,
                                        None, 0, beta, _native.ptr(tC), N, M * N, _native.stream_ptr()), "gemm")
    assert rel(tC.cpu().numpy(), alpha * A @ Bm + beta * C) < 1e-14


def test_dgemm_row_gather():
    lib = _native.load()
    rng = np.random.default_rng(1)
    M, N, K, B = 48, 64, 32, 3
    U = rng.standard_normal((500, N))
    idx = np.stack([rng.integers(0, 500, K) for _ in range(B)]).astype(np.int32)
    A = rng.standard_normal((B, M, K))
    tA, tU, ti = cuda(A), cuda(U), cuda(idx)
    tC = torch.zeros((B, M, N), dtype=torch.float64, device="cuda")
    _native.check(lib.hps_dgemm_batched(_native.context(), M, N, K, B, 1.0, _native.ptr(tA), K, M * K, _native.ptr(tU), N, 0,
                                        _native.ptr(ti), K, 0.0, _native.ptr(tC), N, M * N, _native.stream_ptr()), "g")
    want = np.stack([A[b] @ U[idx[b]] for b in range(B)])
    assert rel(tC.cpu().numpy(), want) < 1e-14


@pytest.mark.parametrize("M,N,K,B", [(21, 7, 21, 3), (84, 84, 42, 2), (5, 3, 7, 1), (130, 66, 33, 4)])
def test_dgemm_generic_shapes(M, N, K, B):
    """Shapes the vectorised path cannot take (K % 16, odd N / leading dims) use the generic path."""
    lib = _native.load()
    rng = np.random.default_rng(M * N + K)
    A, Bm, C = rng.standard_normal((B, M, K)), rng.standard_normal((B, K, N)), rng.standard_normal((B, M, N))
    tA, tB, tC = cuda(A), cuda(Bm), cuda(C)
    _native.check(lib.hps_dgemm_batched(_native.context(), M, N, K, B, 1.5, _native.ptr(tA), K, M * K, _native.ptr(tB), N, K * N, None, 0,
                                        -0.5, _native.ptr(tC), N, M * N, _native.stream_ptr()), "gemm")
    assert rel(tC.cpu().numpy(), 1.5 * A @ Bm - 0.5 * C) < 1e-14


def test_dgemm_rejects_empty_k():
    lib = _native.load()
    t = torch.zeros(64, dtype=torch.float64, device="cuda")
    st = lib.hps_dgemm_batched(_native.context(), 4, 4, 0, 1, 1.0, _native.ptr(t), 4, 0, _native.ptr(t), 4, 0, None, 0, 0.0,
                               _native.ptr(t), 4, 0, _native.stream_ptr())
    assert st == _native.HPS_ERR_ARG


@pytest.mark.parametrize("nb,n3,ne,ldu,nrhs", [(1, 32, 128, 1, 1), (2, 16, 96, 1, 1), (2, 16, 96, 8, 3),
                                               (4, 32, 128, 16, 16), (3, 64, 256, 64, 64)])
def test_solve_level(nb, n3, ne, ldu, nrhs):
    lib = _native.load()
    rng = np.random.default_rng(nb * n3)
    N = 300 + nb * n3
    S = rng.standard_normal((nb, n3, ne))
    Ie = np.stack([rng.permutation(300)[:ne] for _ in range(nb)]).astype(np.int32)
    u = np.zeros((N, ldu))
    u[:300] = rng.standard_normal((300, ldu))
    tS, tI, tu = cuda(S), cuda(Ie), cuda(u)
    _native.check(lib.hps_solve_level(_native.context(), nb, n3, ne, _native.ptr(tS), _native.ptr(tI), 300, _native.ptr(tu), ldu,
                                      nrhs, _native.stream_ptr()), "solve")
    ref = u.copy()
    for b in range(nb):
        ref[300 + b * n3:300 + (b + 1) * n3, :nrhs] = S[b] @ u[Ie[b], :nrhs]
    assert rel(tu.cpu().numpy()[:, :nrhs], ref[:, :nrhs]) < 1e-14


def _host_fields(kind, n_leaf=1024, row=256, seed=0):
    rng = np.random.default_rng(seed)
    if kind == "distinct":
        return {"c11": rng.standard_normal((n_leaf, row)), "c22": rng.standard_normal((n_leaf, row))}
    if kind == "duplicates":  # 37 distinct rows scattered over the leaves, one field
        base = rng.standard_normal((37, row))
        return {"c": base[rng.integers(0, 37, n_leaf)]}
    # two fields whose duplicate patterns differ: leaves group only where both agree
    a, b = rng.standard_normal((5, row)), rng.standard_normal((3, row))
    ia, ib = rng.integers(0, 5, n_leaf), rng.integers(0, 3, n_leaf)
    f = {"c11": a[ia], "c1": b[ib]}
    f["c11"][7] = -0.0 * f["c11"][7]  # signed zeros / bit patterns differ from +0.0
    return f


@pytest.mark.parametrize("kind", ["distinct", "duplicates", "mixed"])
def test_device_grouping_matches_host(kind):
    from paper_1307_2665_b200 import solver
    fields = _host_fields(kind)
    n_leaf = next(iter(fields.values())).shape[0]
    full = dict.fromkeys(solver.COEFF_NAMES, 0.0)
    full.update(fields)
    reps_h, gid_h = solver._group(full, n_leaf)
    dev = [cuda(full[n]) for n in solver.COEFF_NAMES if not np.isscalar(full[n])]
    reps_d, gid_d = solver._group_device(dev, n_leaf)
    assert np.array_equal(reps_d.cpu().numpy(), reps_h)
    assert np.array_equal(gid_d.cpu().numpy(), gid_h)


def test_leaf_verify_flags_a_wrong_representative():
    import ctypes
    lib = _native.load()
    f = cuda(np.arange(4 * 256, dtype=np.float64).reshape(4, 256))
    ptrs = (ctypes.c_void_p * 1)(_native.ptr(f).value)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    ok = torch.tensor([0, 1, 2, 3], dtype=torch.int64, device="cuda")
    _native.check(lib.hps_leaf_verify(4, 256, 1, ptrs, _native.ptr(ok), _native.ptr(flag), _native.stream_ptr()), "v")
    assert int(flag.item()) == 0
    wrong = torch.tensor([0, 0, 2, 3], dtype=torch.int64, device="cuda")
    _native.check(lib.hps_leaf_verify(4, 256, 1, ptrs, _native.ptr(wrong), _native.ptr(flag), _native.stream_ptr()), "v")
    assert int(flag.item()) == 1


def test_two_contexts_on_one_device():
    """Two hps_ctx_t on one device: independent options and split-K scratch; concurrent split-K
    GEMMs on two streams through the two contexts give the same bits as alone."""
    lib = _native.load()
    a, b = _native.Context(0), _native.Context(0)
    try:
        assert lib.hps_ctx_device(a) == 0 and lib.hps_ctx_device(b) == 0
        b.set("splitk", 0)
        assert a.get("splitk") == 1 and b.get("splitk") == 0
        rng = np.random.default_rng(3)
        M, N, K = 128, 128, 4096  # 4 tiles: split-K in a context that allows it
        A, B = cuda(rng.standard_normal((M, K))), cuda(rng.standard_normal((K, N)))
        outs = []
        for cx in (a, b):
            C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
            _native.check(lib.hps_dgemm_batched(cx, M, N, K, 1, 1.0, _native.ptr(A), K, 0, _native.ptr(B), N, 0, None,
                                                0, 0.0, _native.ptr(C), N, 0, _native.stream_ptr()), "gemm")
            outs.append(C)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        conc = [torch.zeros((M, N), dtype=torch.float64, device="cuda") for _ in range(2)]
        torch.cuda.synchronize()
        for cx, s, C in ((a, s1, conc[0]), (b, s2, conc[1])):
            with torch.cuda.stream(s):
                _native.check(lib.hps_dgemm_batched(cx, M, N, K, 1, 1.0, _native.ptr(A), K, 0, _native.ptr(B), N, 0,
                                                    None, 0, 0.0, _native.ptr(C), N, 0, _native.stream_ptr(s)), "g")
        torch.cuda.synchronize()
        assert torch.equal(conc[0], outs[0]) and torch.equal(conc[1], outs[1])
        want = A.cpu().numpy() @ B.cpu().numpy()
        assert rel(outs[0].cpu().numpy(), want) < 1e-13 and rel(outs[1].cpu().numpy(), want) < 1e-13
    finally:
        a.close()
        b.close()


def test_lookahead_refuses_odd_batch():
    """hps_merge_level_ahead with parent arguments but an odd nbatch returns HPS_ERR_ARG instead of
    skipping the look-ahead the caller relies on."""
    lib = _native.load()
    n3, ne, q = 32, 128, 16
    m = ne // 2 + n3
    T = torch.zeros((6, m, m), dtype=torch.float64, device="cuda")
    maps = torch.zeros(ne + 2 * n3, dtype=torch.int32, device="cuda")
    vm = torch.zeros(2 * q, dtype=torch.float64, device="cuda")
    S = torch.empty((3, n3, ne), dtype=torch.float64, device="cuda")
    To = torch.empty((3, ne, ne), dtype=torch.float64, device="cuda")
    wsb = lib.hps_merge_workspace_bytes(3, n3, ne)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    pwsb = lib.hps_merge_workspace_bytes(2, 64, 256)
    pws = torch.empty(pwsb, dtype=torch.uint8, device="cuda")
    st = torch.full((2,), -1, dtype=torch.int32, device="cuda")
    pmaps = torch.zeros(256 + 128, dtype=torch.int32, device="cuda")
    r = lib.hps_merge_level_ahead(_native.context(), 3, n3, ne, m, q, _native.ptr(T), m * m, None, _native.ptr(maps),
                                  _native.ptr(vm), _native.ptr(S), _native.ptr(To), _native.ptr(ws), wsb,
                                  _native.ptr(st), 0, 0, _native.ptr(pmaps), 64, 256, _native.ptr(vm), _native.ptr(pws),
                                  pwsb, _native.ptr(st), 0, 0, _native.stream_ptr())
    assert r == _native.HPS_ERR_ARG and "even nbatch" in _native.last_error()


@pytest.mark.parametrize("scheme,count", [("slices", 8), ("slices", 6), ("moduli", 14), ("moduli", 12)])
@pytest.mark.parametrize("M,N,K,B", [(512, 768, 256, 1), (1024, 256, 512, 3), (256, 4096, 1024, 2)])
def test_emulated_dgemm_accuracy(M, N, K, B, scheme, count):
    """FP64 GEMM on the int8 tensor cores (emu.cu): with 8 slices or 14 moduli the error is at or
    below the DMMA GEMM's against an exact (long double) reference, with rows / columns spanning 16
    decades; with 6 slices or 12 moduli it is within 2^-40 of the row x column scale."""
    lib = _native.load()
    rng = np.random.default_rng(M + N + K + count)
    A = rng.standard_normal((B, M, K)) * 10.0 ** rng.uniform(-8, 8, (B, M, 1))
    Bm = rng.standard_normal((B, K, N)) * 10.0 ** rng.uniform(-8, 8, (B, 1, N))
    exact = np.einsum("bmk,bkn->bmn", A.astype(np.longdouble), Bm.astype(np.longdouble))
    scale = np.abs(A).max(axis=2)[:, :, None] * np.abs(Bm).max(axis=1)[:, None, :] * K
    errs = {}
    opts = {"dmma": dict(emu_slices=0, emu_moduli=0),
            "emu": dict(emu_slices=count, emu_moduli=0) if scheme == "slices" else dict(emu_slices=0, emu_moduli=count)}
    for name, o in opts.items():
        cx = _native.Context(0, emu_min_work=1, emu_min_k=16, **o)
        try:
            tA, tB = cuda(A), cuda(Bm)
            tC = torch.zeros((B, M, N), dtype=torch.float64, device="cuda")
            n0 = lib.hps_launch_count()
            _native.check(lib.hps_dgemm_batched(cx, M, N, K, B, 1.0, _native.ptr(tA), K, M * K, _native.ptr(tB), N,
                                                K * N, None, 0, 0.0, _native.ptr(tC), N, M * N, _native.stream_ptr()),
                          "gemm")
            torch.cuda.synchronize()
            launches = lib.hps_launch_count() - n0
            errs[name] = float((np.abs(tC.cpu().numpy() - exact) / scale).max())
        finally:
            cx.close()
        if name == "emu":
            assert launches >= 5, launches  # the emulated path ran (scales, residues / digits, products, accumulation)
    print(f"M={M} N={N} K={K}: max error / (K max|a_i| max|b_j|): DMMA {errs['dmma']:.2e}, "
          f"emulated ({count} {scheme}) {errs['emu']:.2e}")
    if count in (8, 14):
        assert errs["emu"] <= max(2 * errs["dmma"], 2.0 ** -52), errs
    else:
        assert errs["emu"] <= 2.0 ** -40, errs


@pytest.mark.parametrize("moduli", [13, 14, 15, 16])
def test_emulated_dgemm_nonfinite_and_panels(moduli):
    """Modular emulation: output column panels (a small scratch cap forces several), the merge's
    alpha, a non-finite row (NaN row of the output, flagged like the DMMA path) and zero rows."""
    lib = _native.load()
    M, N, K, B = 256, 1040, 512, 2
    rng = np.random.default_rng(moduli)
    A = rng.standard_normal((B, M, K))
    Bm = rng.standard_normal((B, K, N))
    A[1, 5, 7] = np.inf
    A[0, 9, :] = 0.0
    exact = np.einsum("bmk,bkn->bmn", A.astype(np.longdouble), Bm.astype(np.longdouble)) * -2.0
    cx = _native.Context(0, emu_min_work=1, emu_min_k=16, emu_slices=0, emu_moduli=moduli, emu_scratch_mb=1)
    try:
        tA, tB = cuda(A), cuda(Bm)
        tC = torch.zeros((B, M, N), dtype=torch.float64, device="cuda")
        _native.check(lib.hps_dgemm_batched(cx, M, N, K, B, -2.0, _native.ptr(tA), K, M * K, _native.ptr(tB), N,
                                            K * N, None, 0, 0.0, _native.ptr(tC), N, M * N, _native.stream_ptr()),
                      "gemm")
        C = tC.cpu().numpy()
    finally:
        cx.close()
    assert np.isnan(C[1, 5]).all()
    assert (C[0, 9] == 0.0).all()
    ok = np.ones(C.shape, bool)
    ok[1, 5] = False
    scale = np.abs(A[..., :]).max(axis=2)[:, :, None] * np.abs(Bm).max(axis=1)[:, None, :] * K
    scale[1, 5] = 1.0
    scale[0, 9] = 1.0
    err = float((np.abs(C - exact)[ok] / scale[ok]).max())
    assert err <= 2.0 ** -50, err


@pytest.mark.parametrize("M,N,K,B,mb", [(200, 544, 272, 3, 8192), (200, 544, 272, 3, 1), (1024, 1024, 1024, 2, 8192),
                                        (384, 4096, 2048, 1, 8192), (130, 96, 1040, 5, 8192)])
def test_emulated_dgemm_engines_bitwise(M, N, K, B, mb):
    """Modular emulation: the hand-written tcgen05 int8 kernels (TMA, TMEM accumulators, residues
    reduced in the epilogue; single CTAs = engine 0, CTA pairs = engine 2) and cuBLASLt's IMMA GEMM
    (engine 1) compute the same exact integer residues, so the reconstructed FP64 products are
    bitwise equal; partial tiles in M, N and K, batches and output column panels (mb: scratch cap in
    MB) included."""
    lib = _native.load()
    rng = np.random.default_rng(M * N + K)
    A = rng.standard_normal((B, M, K)) * 10.0 ** rng.uniform(-4, 4, (B, M, 1))
    Bm = rng.standard_normal((B, K, N))
    out = {}
    for engine in (0, 1, 2):
        cx = _native.Context(0, emu_min_work=1, emu_min_k=16, emu_slices=0, emu_moduli=14, emu_engine=engine,
                             emu_scratch_mb=mb)
        try:
            tA, tB = cuda(A), cuda(Bm)
            tC = torch.zeros((B, M, N), dtype=torch.float64, device="cuda")
            _native.check(lib.hps_dgemm_batched(cx, M, N, K, B, 1.0, _native.ptr(tA), K, M * K, _native.ptr(tB), N,
                                                K * N, None, 0, 0.0, _native.ptr(tC), N, M * N, _native.stream_ptr()),
                          "gemm")
            torch.cuda.synchronize()
            out[engine] = tC.cpu().numpy()
        finally:
            cx.close()
    exact = np.einsum("bmk,bkn->bmn", A.astype(np.longdouble), Bm.astype(np.longdouble))
    scale = np.abs(A).max(axis=2)[:, :, None] * np.abs(Bm).max(axis=1)[:, None, :] * K
    err = float((np.abs(out[0] - exact) / scale).max())
    print(f"M={M} N={N} K={K} B={B}: tcgen05 single / pair vs cuBLASLt max |diff| {np.abs(out[0] - out[1]).max():.1e} "
          f"/ {np.abs(out[2] - out[1]).max():.1e}, error {err:.2e}")
    assert np.array_equal(out[0], out[1])
    assert np.array_equal(out[2], out[1])
    assert err <= 2.0 ** -52


@pytest.mark.parametrize("engine", [0, 2])
@pytest.mark.parametrize("M,N,nc,j0,K,batch,nmod", [(300, 640, 320, 256, 1040, 2, 3), (128, 256, 256, 0, 128, 1, 14),
                                                   (520, 1024, 512, 512, 4096, 1, 2), (64, 96, 64, 32, 16, 3, 4)])
def test_i8gemm_mod_exact(engine, M, N, nc, j0, K, batch, nmod):
    """The tcgen05 int8 kernel through the C ABI against exact int64 products: every residue
    ((A B^T) mod m) + 128 bitwise, for partial tiles in M / N / K, an output column panel at j0,
    several moduli x batches, both the single-CTA and the CTA-pair kernel."""
    import ctypes

    lib = _native.load()
    rng = np.random.default_rng(M + N + K + nmod)
    moduli = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199][:nmod]
    nz = nmod * batch
    A = rng.integers(-128, 128, (nz, M, K), dtype=np.int8)
    B = rng.integers(-128, 128, (nz, N, K), dtype=np.int8)
    tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    tR = torch.zeros((nz, M, nc), dtype=torch.uint8, device="cuda")
    mods = (ctypes.c_int * nmod)(*moduli)
    _native.check(lib.hps_i8gemm_mod(_native.context(), _native.ptr(tA), _native.ptr(tB), _native.ptr(tR), M, N, nc, j0,
                                     K, nz, batch, mods, nmod, engine, _native.stream_ptr()), "i8gemm")
    R = tR.cpu().numpy()
    for z in range(nz):
        m = moduli[z // batch]
        C = A[z].astype(np.int64) @ B[z, j0:j0 + nc].astype(np.int64).T
        r = np.mod(C, m)
        r = np.where(r > 127, r - m, r) + 128
        assert np.array_equal(R[z], r.astype(np.uint8)), (z, m)


def test_i8gemm_mod_rejects_bad_arguments():
    import ctypes

    lib = _native.load()
    mods = (ctypes.c_int * 2)(256, 255)
    t = torch.zeros(1 << 16, dtype=torch.int8, device="cuda")
    r = lib.hps_i8gemm_mod(_native.context(), _native.ptr(t), _native.ptr(t), _native.ptr(t), 16, 64, 48, 0, 32, 2, 1,
                           mods, 2, 0, _native.stream_ptr())  # nc % 32 != 0
    assert r == _native.HPS_ERR_ARG and "unsupported" in _native.last_error()


@pytest.mark.parametrize("moduli", [6, 13, 14, 15, 16])
@pytest.mark.parametrize("M,N,K,B", [(200, 544, 272, 2), (132, 100, 1040, 3), (512, 512, 4096, 1)])
def test_emulated_dgemm_split_paths_bitwise(M, N, K, B, moduli):
    """Modular emulation: the operand residues computed on the integer pipes (int64 conversion, a
    small int8 MMA per element pair, integer reduction; HPS_OPT_EMU_SPLIT 1) are the same signed
    bytes as the FP64-pipe ones (0), so the products are bitwise equal; partial tiles in M, N and K,
    every leftover count of moduli (NM % 4), scales spread over 40 binades."""
    lib = _native.load()
    rng = np.random.default_rng(M + moduli)
    A = rng.standard_normal((B, M, K)) * np.exp2(rng.integers(-20, 20, (B, M, 1)))
    Bm = rng.standard_normal((B, K, N)) * np.exp2(rng.integers(-20, 20, (B, 1, N)))
    A[0, 3, :] = 0.0
    outs = []
    for split in (0, 1):
        cx = _native.Context(0, emu_min_work=1, emu_min_k=16, emu_slices=0, emu_moduli=moduli, emu_split=split)
        try:
            tA, tB = cuda(A), cuda(Bm)
            tC = torch.zeros((B, M, N), dtype=torch.float64, device="cuda")
            _native.check(lib.hps_dgemm_batched(cx, M, N, K, B, 1.0, _native.ptr(tA), K, M * K, _native.ptr(tB), N,
                                                K * N, None, 0, 0.0, _native.ptr(tC), N, M * N, _native.stream_ptr()),
                          "gemm")
            outs.append(tC.cpu().numpy())
        finally:
            cx.close()
    assert np.array_equal(outs[0], outs[1])
    ref = np.einsum("bmk,bkn->bmn", A, Bm)
    scale = np.abs(A).max(axis=2)[:, :, None] * np.abs(Bm).max(axis=1)[:, None, :] * K
    scale[0, 3] = 1.0
    assert float((np.abs(outs[1] - ref) / scale).max()) <= (2.0 ** -50 if moduli >= 13 else 2.0 ** -10)


def test_emulated_dgemm_extreme_scales():
    """Modular emulation: rows / columns near the fp64 range edges (1e-300, 1e+300 and subnormal
    entries) take the rescaled norm path and still give DGEMM-level relative errors."""
    lib = _native.load()
    rng = np.random.default_rng(7)
    M, N, K = 64, 128, 256
    A = rng.standard_normal((1, M, K))
    Bm = rng.standard_normal((1, K, N))
    A[0, 0] *= 1e-300
    A[0, 1] *= 1e+290
    A[0, 2, :8] = 5e-324  # subnormal entries
    Bm[0, :, 3] *= 1e-200
    Bm[0, :, 4] *= 1e+200
    exact = np.einsum("bmk,bkn->bmn", A.astype(np.longdouble), Bm.astype(np.longdouble))
    cx = _native.Context(0, emu_min_work=1, emu_min_k=16, emu_slices=0, emu_moduli=14)
    try:
        tA, tB = cuda(A), cuda(Bm)
        tC = torch.zeros((1, M, N), dtype=torch.float64, device="cuda")
        _native.check(lib.hps_dgemm_batched(cx, M, N, K, 1, 1.0, _native.ptr(tA), K, M * K, _native.ptr(tB), N, K * N,
                                            None, 0, 0.0, _native.ptr(tC), N, M * N, _native.stream_ptr()), "gemm")
        C = tC.cpu().numpy().astype(np.longdouble)
    finally:
        cx.close()
    scale = np.abs(A).max(axis=2)[:, :, None].astype(np.longdouble) * np.abs(Bm).max(axis=1)[:, None, :] * K
    ok = (scale > 1e-290) & (scale < 1e300)  # results representable in fp64 without underflow / overflow
    err = np.abs(C - exact)[ok] / scale[ok]
    assert np.isfinite(C[0, 1, :3]).all() and np.isfinite(C[0, 0]).all()
    assert float(err.max()) <= 2.0 ** -50, float(err.max())
