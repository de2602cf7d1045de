"""Algorithmic work model of the hot path: flop and minimum-byte counts per stage,
used by bench.py's roofline. Standard LAPACK counts; leaf work is per distinct coefficient group,
as in the reference (solver.py:208-246)."""


def depth_sizes(L, q, d):
    """(n3, ne) of every parent at depth d (0 = root) of a 4^L-leaf tree with q Gauss nodes per
    leaf side: even depths split vertically (square parents), odd depths horizontally."""
    j = d // 2
    if d % 2 == 0:
        side = 2 ** (L - j)
        return side * q, 4 * side * q
    w, h = 2 ** (L - j - 1), 2 ** (L - j)
    return w * q, 2 * (w + h) * q


def leaf_flops(p):
    """Per group: LU of A_ii, solve for the n_b + 1 right-hand sides (A_ie and the probe),
    T1 = L43i Psi and T = T1 L1."""
    ni, nb, ng = (p - 2) ** 2, 4 * (p - 1), 4 * p
    return 2.0 / 3.0 * ni ** 3 + 2.0 * ni ** 2 * (nb + 1) + 2.0 * ng * ni * nb + 2.0 * ng * nb * ng


def leaf_bytes(p, nfields=6):
    """Per group: coefficient samples in, T and Psi out."""
    ni, nb, ng = (p - 2) ** 2, 4 * (p - 1), 4 * p
    return 8.0 * (nfields * p * p + ng * ng + ni * nb)


def merge_flops_depth(L, q, d):
    n3, ne = depth_sizes(L, q, d)
    return (2 ** d) * (2.0 / 3.0 * n3 ** 3 + 2.0 * n3 ** 2 * ne + 2.0 * n3 * ne ** 2)


def merge_stage_flops(L, q, ahead=()):
    """Per merge stage (depth d) flops as executed: a depth in `ahead` (solver.lookahead_depths)
    also runs its parent's interface inverse (2/3 n3^3 per parent, moved from depth d - 1) and the
    look-ahead GEMM that forms the parent's X (4 pn3^2 n3 per parent, extra work beyond the
    reference count, so not added: achieved rates stay on the algorithmic count)."""
    out = {d: merge_flops_depth(L, q, d) for d in range(2 * L)}
    for d in ahead:
        pn3, _ = depth_sizes(L, q, d - 1)
        inv = (2 ** (d - 1)) * 2.0 / 3.0 * pn3 ** 3
        out[d - 1] -= inv
        out[d] += inv
    return out


def merge_bytes_depth(L, q, d):
    """Children's T in (two m x m, m = ne/2 + n3), S and T out."""
    n3, ne = depth_sizes(L, q, d)
    m = ne // 2 + n3
    return (2 ** d) * 8.0 * (2 * m * m + n3 * ne + ne * ne)


def solve_flops(L, q, b):
    return 2.0 * b * sum((2 ** d) * depth_sizes(L, q, d)[0] * depth_sizes(L, q, d)[1] for d in range(2 * L))


def solve_S_bytes(L, q):
    return 8.0 * sum((2 ** d) * depth_sizes(L, q, d)[0] * depth_sizes(L, q, d)[1] for d in range(2 * L))


def build_roofline_seconds(L, q, ngroups, f64_tflops, hbm_gbs):
    """t_roof = sum over stages of max(flop / FP64 peak, bytes / HBM peak)."""
    F, B = f64_tflops * 1e12, hbm_gbs * 1e9
    t = max(ngroups * leaf_flops(q) / F, ngroups * leaf_bytes(q) / B)
    for d in range(2 * L):
        t += max(merge_flops_depth(L, q, d) / F, merge_bytes_depth(L, q, d) / B)
    return t


def emulated_gemms(L, q, d, min_k=512, min_work=2 ** 32):
    """(M, N, K, batch) of the merge GEMMs of depth d that run as the FP64 emulation on int8
    (csrc/emu.cu: K >= min_k and M N K batch >= min_work): S = X^-1 R (n3 x ne x n3) and
    T = blk + C S (ne x ne x n3), 2^d merges."""
    n3, ne = depth_sizes(L, q, d)
    out = []
    for M, N, K in ((n3, ne, n3), (ne, ne, n3)):
        if K >= min_k and float(M) * N * K * 2 ** d >= min_work and M % 4 == 0 and N % 4 == 0 and K % 16 == 0:
            out.append((M, N, K, 2 ** d))
    return out


def emulated_int8_ops(L, q, d, products, **kw):
    """int8 tensor operations of depth d's emulated GEMMs: `products` int8 products of 2 M N K each
    (the modular scheme: one per modulus; the slice scheme: s (s + 1) / 2)."""
    if products <= 0:
        return 0.0
    return sum(products * 2.0 * M * N * K * b for M, N, K, b in emulated_gemms(L, q, d, **kw))
