"""Host-side logic of the product path that runs without a GPU: coefficient sampling and leaf
grouping (solver.py:196-222), geometry constants, problem generators, memory accounting."""
import numpy as np
import pytest

import paper_1307_2665_b200 as P
from oracle import hps_oracle as O
from paper_1307_2665_b200 import problems, solver
from paper_1307_2665_b200.grid import layout_of

from _util import coeff_dict


@pytest.mark.parametrize("cfg,L", [(1, 3), (2, 3), (4, 4), (5, 2)])
def test_grouping_matches_reference_semantics(cfg, L):
    co = problems.coefficients(cfg)
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
    lay = layout_of(tree)
    geom = P.LeafGeometry.get(16, tree.leaf_width, tree.leaf_height)
    fields = solver._sample(co, lay, geom)
    reps, gid = solver._group(fields, 4 ** L)
    ot = O.build_tree((0, 1, 0, 1), L, 16)
    og = O.Geometry(16, ot.leaf_width, ot.leaf_height)
    ofields = O.sample_coefficients(coeff_dict(co), ot, og)
    oreps, ogid = O.group_leaves(ofields, 4 ** L)
    assert np.array_equal(reps, oreps) and np.array_equal(gid, ogid)
    for name in O.COEFF_NAMES:
        if not np.isscalar(fields[name]):
            assert np.array_equal(fields[name], ofields[name])


def test_var_helmholtz_groups_collapse_bitwise_equal_leaves():
    # cfg 4's symmetric coefficient makes some leaves bitwise equal (61,086 of 65,536 at L=8)
    co = problems.coefficients(4)
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 5, 16)
    geom = P.LeafGeometry.get(16, tree.leaf_width, tree.leaf_height)
    reps, gid = solver._group(solver._sample(co, layout_of(tree), geom), 4 ** 5)
    assert reps.size < 4 ** 5 and gid.max() == reps.size - 1 and np.all(reps[gid[reps]] == reps)


def test_device_constants_layout():
    g = P.LeafGeometry.get(16, 1 / 64, 1 / 64)
    blob, idx, pmax = g.device_constants()
    p2, ni, nb, ng = 256, 196, 60, 64
    assert blob.size == 4 * p2 + ng * nb + ng * ni + nb * ng + ni
    assert np.array_equal(blob[:p2], g.Dx.ravel())
    assert np.array_equal(blob[2 * p2:3 * p2], (g.Dx @ g.Dx).ravel())
    assert np.array_equal(idx[:ni], g.J_i) and np.array_equal(idx[ni:], g.J_e)
    assert pmax == np.abs(blob[-ni:]).max()


@pytest.mark.parametrize("axis", ["v", "h"])
def test_corner_modes_are_null_vectors_of_the_interface(axis):
    """X V = 0 and [T13a; T23b] V = 0 for the analytic corner modes (the deflation basis)."""
    L = 2
    co = problems.coefficients(2)
    ot = O.build_tree((0, 1, 0, 1), L, 16)
    st = O.build(ot, coeff_dict(co), keep_T=True)
    geom = P.LeafGeometry.get(16, ot.leaf_width, ot.leaf_height)
    box = 0 if axis == "v" else 1
    a, c = ot.child_a[box], ot.child_b[box]
    j1a, j2b, j3a, j3b = O.split_indices(ot.I_e[a], ot.I_e[c], ot.I_i[box])
    Ta, Tb = st.T[a], st.T[c]
    X = Ta[np.ix_(j3a, j3a)] - Tb[np.ix_(j3b, j3b)]
    C = np.concatenate([Ta[np.ix_(j1a, j3a)], Tb[np.ix_(j2b, j3b)]])
    vs, ve = geom.corner_mode_vectors(axis)
    n3 = X.shape[0]
    m = n3 // 16
    V = np.zeros((n3, m - 1))
    for s in range(m - 1):
        V[s * 16:(s + 1) * 16, s] = ve
        V[(s + 1) * 16:(s + 2) * 16, s] = vs
    assert np.abs(X @ V).max() < 1e-13 * np.abs(X).max()
    assert np.abs(C @ V).max() < 1e-13 * np.abs(C).max()
    Xd = X + np.abs(np.diag(X)).max() * V @ V.T
    assert np.linalg.cond(Xd) < 1e4  # deflated interface is well conditioned


def test_boundary_data_generators():
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 2, 16)
    pts = nodes.points[tree.root.I_e]
    F = problems.boundary_data(2, pts, seed=5, batch=3)
    assert F.shape == (pts.shape[0], 3)
    assert np.array_equal(F, problems.boundary_data(2, pts, seed=5, batch=3))
    t = problems.perimeter_parameter(pts[:, 0], pts[:, 1])
    assert t.min() >= 0 and t.max() < 4
    f1 = problems.boundary_data(1, pts)
    assert f1.shape == (pts.shape[0],) and np.allclose(f1, np.exp(pts[:, 0]) * np.sin(pts[:, 1]))
    F3 = problems.boundary_data(3, pts, seed=2, batch=2)
    U3 = problems.exact_solution(3, pts[:, 0], pts[:, 1], seed=2, batch=2)
    assert np.array_equal(F3, U3)


def test_unknowns_definition():
    assert O.unknowns(6, 16) == 1048576 and O.unknowns(9, 16) == 67108864


def test_work_model_matches_oracle_counts():
    # bench.py's roofline uses paper_1307_2665_b200.work (no oracle import on the measured path);
    # it must agree with the oracle's LAPACK-count restatement
    from paper_1307_2665_b200 import work as W
    for L in (2, 4, 6, 9):
        for d in range(2 * L):
            assert W.depth_sizes(L, 16, d) == O.depth_sizes(L, 16, d)
        assert abs(sum(W.merge_flops_depth(L, 16, d) for d in range(2 * L)) - O.merge_flops(L, 16)) < 1e-6 * O.merge_flops(L, 16)
        assert abs(W.solve_flops(L, 16, 64) - O.solve_flops(L, 16, 64)) < 1.0
    assert W.leaf_flops(16) == O.leaf_flops(16)
    # SURVEY.md §8d build totals: cfg2 1.79e11 flop
    tot = 4096 * W.leaf_flops(16) + sum(W.merge_flops_depth(6, 16, d) for d in range(12))
    assert abs(tot - 1.79e11) / 1.79e11 < 0.01


def test_lookahead_rule_and_stage_flop_accounting(monkeypatch):
    # hps_merge_level_ahead is used where the parent's interface inverse is a latency chain worth
    # hiding: pn3 >= 128 and pn3 * n3 * P <= 3.2e6 (every depth of L <= 7, none at L >= 8). The
    # bench attributes the moved inverse flops to the depth that runs them; totals are unchanged.
    from paper_1307_2665_b200 import work as W
    monkeypatch.delenv("HPS_AHEAD_MIN_N3", raising=False)
    monkeypatch.delenv("HPS_AHEAD_WORK", raising=False)
    for L, want in ((4, {1, 2, 3}), (6, set(range(1, 8))), (7, set(range(1, 10))), (8, set()), (9, set())):
        tree, _ = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
        lay = layout_of(tree)
        got = solver.lookahead_depths(lay)
        assert got == want, (L, got)
        f = W.merge_stage_flops(L, 16, got)
        ref = {d: W.merge_flops_depth(L, 16, d) for d in range(2 * L)}
        assert abs(sum(f.values()) - sum(ref.values())) < 1e-6 * sum(ref.values())
        inv = {d: 2 ** d * 2.0 / 3.0 * W.depth_sizes(L, 16, d)[0] ** 3 for d in range(2 * L)}
        for d in range(2 * L):  # depth d's inverse runs in depth d + 1 when d + 1 looks ahead
            want_d = ref[d] - (inv[d] if d + 1 in got else 0.0) + (inv[d - 1] if d in got else 0.0)
            assert f[d] == pytest.approx(want_d)
    monkeypatch.setenv("HPS_AHEAD_MIN_N3", "0")
    tree, _ = P.build_tree(P.Rectangle(0, 1, 0, 1), 6, 16)
    assert solver.lookahead_depths(layout_of(tree)) == set()


@pytest.mark.parametrize("cfg,L", [(3, 4), (4, 4)])
def test_interface_conditioning_report(cfg, L):
    """Helmholtz interfaces (configs 3, 4) at every depth with n3 > q: cond of the deflated X_d, cond of
    its leading half block A11 (what a factorisation pivoting only inside blocks depends on) and the
    growth factor max|U| / max|X_d| of LAPACK's partially pivoted LU (what the device LU depends on;
    tests/test_gpu_lu.py checks it picks LAPACK's pivots). Printed with pytest -s."""
    import scipy.linalg as sla
    ot = O.build_tree((0, 1, 0, 1), L, 16)
    st = O.build(ot, {n: getattr(problems.coefficients(cfg), n) for n in O.COEFF_NAMES}, keep_T=True)
    geom = P.LeafGeometry.get(16, ot.leaf_width, ot.leaf_height)
    for d in range(2 * L - 1):
        box = (1 << d) - 1
        axis = "v" if d % 2 == 0 else "h"
        a, c = ot.child_a[box], ot.child_b[box]
        j1a, j2b, j3a, j3b = O.split_indices(ot.I_e[a], ot.I_e[c], ot.I_i[box])
        X = st.T[a][np.ix_(j3a, j3a)] - st.T[c][np.ix_(j3b, j3b)]
        n3 = X.shape[0]
        vs, ve = geom.corner_mode_vectors(axis)
        V = np.zeros((n3, n3 // 16 - 1))
        for s_ in range(n3 // 16 - 1):
            V[s_ * 16:(s_ + 1) * 16, s_] = ve
            V[(s_ + 1) * 16:(s_ + 2) * 16, s_] = vs
        Xd = X + np.abs(np.diag(X)).max() * V @ V.T
        h = n3 // 2
        lu, _ = sla.lu_factor(Xd)
        growth = np.abs(np.triu(lu)).max() / np.abs(Xd).max()
        cx, c11 = np.linalg.cond(Xd), np.linalg.cond(Xd[:h, :h])
        print(f"cfg{cfg} L{L} depth {d}: n3 {n3}, cond(X_d) {cx:.2e}, cond(A11) {c11:.2e}, LU growth {growth:.2f}")
        assert np.isfinite(cx) and cx < 1e10 and growth < 1e3  # cfg4 reaches 5e6 (its global problem is near-resonant)


def test_crt_reconstruction_model():
    """The modular FP64 emulation's reconstruction (csrc/emu.cu, crt_constants / k_crt_accum)
    restated with Python integers and float64: for integers |C'| <= Mod / 8 given by their residues
    modulo the 14 moduli, the exact high sum (run over the biased doubles d = r + 4224 from a
    bias-cancelling start value, as the kernel does), the rounded quotient and the two-part
    correction recover C' to within an ulp of the largest |C'|; the quotient never rounds the
    wrong way and every partial high sum stays an exact integer."""
    import math

    moduli = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199]
    Mod = math.prod(moduli)
    bits = Mod.bit_length()
    E = bits - 36
    bias = 4224.0  # 4096 (the byte-permuted double's leading one) + 128 (the byte's bias)

    def split(v, keep33=False):  # v = hi 2^E + lo, |lo| <= 2^(E-1); keep33: lo to a multiple of 2^(E-34)
        unit = 1 << E
        qv = (v + unit // 2) >> E if v >= 0 else -((-v + unit // 2) >> E)
        rem = v - qv * unit
        if keep33:
            u2 = 1 << (E - 34)
            rem = ((rem + u2 // 2) // u2 if rem >= 0 else -((-rem + u2 // 2) // u2)) * u2
        return qv, rem

    W, wlo = [], []
    for m in moduli:
        Ml = Mod // m
        y = pow(Ml % m, -1, m)
        w = (Ml * y) % Mod
        if w > Mod // 2:
            w -= Mod
        h, lo = split(w, True)
        assert abs(h) <= 2 ** 35 + 1 and abs(lo) <= 2 ** (E - 1)
        W.append(float(h))
        wlo.append(float(lo))
    Mh, Mlo = split(Mod)
    twoE, twoE_over_M, inv_M = 2.0 ** E, 2.0 ** E / float(Mod), 1.0 / float(Mod)
    shi0, slo0 = -bias * sum(W), -bias * sum(wlo)
    assert shi0 == -int(bias) * sum(int(w) for w in W)  # exact
    rng = np.random.default_rng(11)
    bound = Mod // 8
    vals = [int(x) for x in rng.integers(-2 ** 62, 2 ** 62, 200)]
    vals = [v * (bound // 2 ** 62) + int(rng.integers(0, 2 ** 40)) for v in vals] + [bound, -bound, 0, 1, -1]
    for C in vals:
        r = [((C % m) + m // 2) % m - m // 2 for m in moduli]  # symmetric residues, |r| <= 128
        shi, slo = shi0, slo0
        exact = int(shi0)
        for rr, Wl, wl in zip(r, W, wlo):
            d = float(rr) + bias  # 4096 + (r + 128)
            shi = shi + d * Wl  # the product (13 x 36 bits) and the sum are exact, as the kernel's fma
            exact += (rr + int(bias)) * int(Wl)
            assert abs(exact) < 2 ** 53 and shi == float(exact)  # every partial sum exact
            slo += d * wl
        assert shi == float(sum(rr * int(Wl) for rr, Wl in zip(r, W)))
        assert slo == float(sum(rr * int(wl) for rr, wl in zip(r, wlo)))  # the low sum is exact too
        q = round(shi * twoE_over_M + slo * inv_M)
        true_q = (sum(rr * (int(Wl) * 2 ** E + int(wl)) for rr, Wl, wl in zip(r, W, wlo)) - C) / Mod
        assert abs(q - true_q) < 0.25 or q == round(true_q)
        X = shi - q * float(Mh)  # exact
        cp = X * twoE + (slo - q * float(Mlo))
        assert abs(cp - C) <= 2.0 ** (bits - 4 - 52), (C, cp)


def test_residue_reduction_model():
    """The integer-pipe operand residues of the modular emulation (csrc/emu.cu, res_tab / res_words)
    restated with numpy integers: the group shift S is a multiple of every modulus of its group and
    keeps v = y + S inside (0, 2^64) for |y| <= 2^61; the byte sums c = sum d_i (256^i mod m) (the
    int8 MMA) are congruent to v and below 2^18 in magnitude; over that whole range the multiply-high
    quotient with the 2^20 bias equals floor((c + h) / m) and r = c - q m is a signed byte congruent
    to y."""
    import math

    moduli = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]
    rng = np.random.default_rng(5)
    for n in (6, 13, 14, 15, 16):
        for grp in (moduli[:min(n, 8)], moduli[8:n]):
            if not grp:
                continue
            P = math.prod(grp)
            S = P * max(1, (1 << 62) // P)
            assert (1 << 61) <= S <= (1 << 64) - (1 << 61)
            assert all(S % m == 0 for m in grp)
            ys = [int(v) for v in rng.integers(-(1 << 61), 1 << 61, 64)] + [-(1 << 61), 1 << 61, 0, -1, 1]
            for m in grp:
                consts = []
                pw = 1
                for _ in range(8):
                    cc = pw % m
                    consts.append(cc - m if cc >= (m + 1) // 2 else cc)
                    pw = pw * 256 % m
                assert all(-128 <= cc <= 127 for cc in consts)
                for y in ys:
                    v = y + S
                    assert 0 < v < 1 << 64
                    c = sum(((v >> (8 * i)) & 0xFF) * consts[i] for i in range(8))
                    assert abs(c) < 1 << 18 and (c - y) % m == 0
    c = np.arange(-(1 << 18), 1 << 18, dtype=np.int64)
    for m in moduli:
        h, minv = m // 2, (1 << 32) // m + 1
        kq = h * minv + (1 << 20)
        assert kq < 1 << 32
        q = (c * minv + kq) >> 32  # arithmetic shift: floor
        assert np.array_equal(q, (c + h) // m)
        r = c - q * m
        assert r.min() >= -h and r.max() <= m - 1 - h and -128 <= r.min() and r.max() <= 127
