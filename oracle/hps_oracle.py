"""CPU oracle for the HPS build/solve hot path. This is TEST INFRASTRUCTURE, not product code.

This is a numpy/scipy restatement of the reference algorithm
(`/root/reference/pkg/src/hpsolve/{grid,leafops,merge,solver}.py`). Every function cites the
reference lines it follows. The only code allowed to import it is `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference` legs. It is the
checker, never the thing measured or shipped. The product path
(`paper_1307_2665_b200`) never imports it.

Pinning: `tests/golden/*.npz` were produced by importing the reference itself
(`tests/golden/make_golden.py`, run in the build container where `/root/reference` exists).
`tests/test_oracle_golden.py` checks this restatement against those vectors: bit-exact for tree,
index and point layout, and within 1e-13 relative for leaf/merge operators. So the oracle is
**pinned** to the reference.

Arithmetic follows the reference's dense branch (`build(..., switch_threshold=None)`). The leaf
stage uses a batched LAPACK gesv (numpy). The merges use LAPACK getrf/getrs (scipy) and a
BLAS gemm. The oracle therefore reproduces the reference's own null-mode garbage in `S`/raw
`u`; parity is gated on null-mode-invariant quantities only.
"""

from __future__ import annotations

import math
from collections import OrderedDict

import numpy as np
import scipy.linalg as sla

COEFF_NAMES = ("c11", "c12", "c22", "c1", "c2", "c")
RESONANCE_COND = 1e13  # leafops.py:33


# ----------------------------------------------------------------------------------------------
# 1-D nodes and interpolation (grid.py:133-201, leafops.py:70-85)
# ----------------------------------------------------------------------------------------------
def gauss_nodes(q):
    """Gauss-Legendre points by Newton on the Legendre recurrence (grid.py:133-154).

    The flop sequence matches the reference (same initial guess, same recurrence, same stop rule),
    so the nodes come out bitwise identical.
    """
    if q < 1:
        raise ValueError("q must be >= 1")
    if q == 1:
        return np.zeros(1)
    x = -np.cos(np.pi * (4 * np.arange(q) + 3) / (4 * q + 2))
    for _ in range(100):
        pm1 = np.zeros_like(x)
        pk = np.ones_like(x)
        for k in range(q):
            pm1, pk = pk, ((2 * k + 1) * x * pk - k * pm1) / (k + 1)
        step = pk / (q * (x * pk - pm1) / (x * x - 1.0))
        x = x - step
        if np.max(np.abs(step)) < 1e-15:
            break
    return np.sort(x)


def cheb_nodes(p, interval=(-1.0, 1.0)):
    """Chebyshev extreme points on [a, b], ascending, exact endpoints (grid.py:157-167)."""
    a, b = interval
    if p < 2:
        raise ValueError("p must be >= 2")
    if not a < b:
        raise ValueError("empty interval")
    t = np.cos(np.pi * np.arange(p) / (p - 1))[::-1]
    x = 0.5 * (a + b) + 0.5 * (b - a) * t
    x[0] = a
    x[-1] = b
    return x


def interp_matrix(src, dst):
    """Barycentric Lagrange interpolation matrix |dst| x |src| (grid.py:170-201)."""
    src = np.atleast_1d(np.asarray(src, dtype=float))
    dst = np.atleast_1d(np.asarray(dst, dtype=float))
    if src.size == 1:
        return np.ones((dst.size, 1))
    scale = 4.0 / max(src.max() - src.min(), np.finfo(float).tiny)
    dif = (src[:, None] - src[None, :]) * scale
    np.fill_diagonal(dif, 1.0)
    w = 1.0 / np.prod(dif, axis=1)
    d = dst[:, None] - src[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        r = w[None, :] / d
        M = r / np.sum(r, axis=1)[:, None]
    for i, j in zip(*np.nonzero(d == 0.0)):
        M[i, :] = 0.0
        M[i, j] = 1.0
    return M


def cheb_diff_matrix(p, interval=(-1.0, 1.0)):
    """Barycentric Chebyshev differentiation matrix, negative-sum diagonal (leafops.py:70-85)."""
    x = cheb_nodes(p, interval)
    w = np.power(-1.0, np.arange(p))
    w[0] *= 0.5
    w[-1] *= 0.5
    D = np.zeros((p, p))
    for i in range(p):
        o = np.array([j for j in range(p) if j != i])
        D[i, o] = (w[o] / w[i]) / (x[i] - x[o])
        D[i, i] = -np.sum(D[i, o])
    return D


# ----------------------------------------------------------------------------------------------
# Tree / node layout (grid.py:204-322)
# ----------------------------------------------------------------------------------------------
class OracleTree:
    """Plain-array restatement of BoxTree + GlobalNodeSet (grid.py:51-130)."""

    def __init__(self, domain, L, q):
        self.domain = tuple(float(v) for v in domain)
        self.L = L
        self.q = q


def build_tree(domain, L, q):
    """Loop restatement of `build_tree` (grid.py:204-322).

    Returns an OracleTree with per-box lists: cells, level, parent, child_a, child_b,
    split_axis, I_e, I_i, plus points (N,2), on_vertical (N,), n_gamma.
    """
    x_lo, x_hi, y_lo, y_hi = (float(v) for v in domain)
    if not (x_lo < x_hi and y_lo < y_hi):
        raise ValueError("degenerate rectangle")
    if L < 0:
        raise ValueError("L must be >= 0")
    if q < 2:
        raise ValueError("q must be >= 2")
    width, height = x_hi - x_lo, y_hi - y_lo
    n = 1 << L
    xline = x_lo + np.arange(n + 1) * (width / n)  # grid.py:220
    yline = y_lo + np.arange(n + 1) * (height / n)  # grid.py:221
    gx = x_lo + (gauss_nodes(q) + 1.0) * 0.5 * (width / n)  # grid.py:222
    gx = gx - x_lo  # grid.py:223
    gy = (gauss_nodes(q) + 1.0) * 0.5 * (height / n)  # grid.py:224

    t = OracleTree((x_lo, x_hi, y_lo, y_hi), L, q)
    cells = [(0, 0, n, n)]
    level = [0]
    parent = [-1]
    ca_l, cb_l, axis_l = [-1], [-1], ["none"]
    # breadth-first creation, vertical cut at even depth (grid.py:229-248)
    frontier = [0]
    for depth in range(2 * L):
        ax = "v" if depth % 2 == 0 else "h"
        nxt = []
        for b in frontier:
            ix, iy, nx, ny = cells[b]
            if ax == "v":
                kids = ((ix, iy, nx // 2, ny), (ix + nx // 2, iy, nx - nx // 2, ny))
            else:
                kids = ((ix, iy, nx, ny // 2), (ix, iy + ny // 2, nx, ny - ny // 2))
            for which, cc in enumerate(kids):
                idx = len(cells)
                cells.append(cc)
                level.append(depth + 1)
                parent.append(b)
                ca_l.append(-1)
                cb_l.append(-1)
                axis_l.append("none")
                if which == 0:
                    ca_l[b] = idx
                else:
                    cb_l[b] = idx
                nxt.append(idx)
            axis_l[b] = ax
        frontier = nxt

    ids = {}
    pts = []
    vert = []

    def reg(key):
        k = ids.get(key)
        if k is None:
            k = len(pts)
            ids[key] = k
            o, line, seg, g = key
            if o == "h":
                pts.append((xline[seg] + gx[g], yline[line]))
                vert.append(False)
            else:
                pts.append((xline[line], yline[seg] + gy[g]))
                vert.append(True)
        return k

    # outer boundary S, E, N, W (grid.py:270-282)
    for seg in range(n):
        for g in range(q):
            reg(("h", 0, seg, g))
    for seg in range(n):
        for g in range(q):
            reg(("v", n, seg, g))
    for seg in range(n):
        for g in range(q):
            reg(("h", n, seg, g))
    for seg in range(n):
        for g in range(q):
            reg(("v", 0, seg, g))
    n_gamma = len(pts)

    nb = len(cells)
    I_i = [np.zeros(0, dtype=np.intp) for _ in range(nb)]
    for b in range(nb):  # parents' cut-line nodes in box order (grid.py:284-295)
        if ca_l[b] < 0:
            continue
        ix, iy, nx, ny = cells[b]
        if axis_l[b] == "v":
            ln = ix + nx // 2
            keys = [("v", ln, j, g) for j in range(iy, iy + ny) for g in range(q)]
        else:
            ln = iy + ny // 2
            keys = [("h", ln, i, g) for i in range(ix, ix + nx) for g in range(q)]
        I_i[b] = np.array([reg(k) for k in keys], dtype=np.intp)

    I_e = [None] * nb
    for b in range(nb - 1, -1, -1):  # bottom-up exterior lists (grid.py:305-319)
        if ca_l[b] < 0:
            ix, iy, _, _ = cells[b]
            keys = ([("h", iy, ix, g) for g in range(q)] + [("v", ix + 1, iy, g) for g in range(q)]
                    + [("h", iy + 1, ix, g) for g in range(q)] + [("v", ix, iy, g) for g in range(q)])
            I_e[b] = np.array([ids[k] for k in keys], dtype=np.intp)
        else:
            sh = set(I_i[b].tolist())
            a, c = I_e[ca_l[b]], I_e[cb_l[b]]
            I_e[b] = np.concatenate([a[[v not in sh for v in a.tolist()]],
                                     c[[v not in sh for v in c.tolist()]]])

    t.cells = cells
    t.level = level
    t.parent = parent
    t.child_a = ca_l
    t.child_b = cb_l
    t.split_axis = axis_l
    t.I_e = I_e
    t.I_i = I_i
    t.points = np.array(pts, dtype=float)
    t.on_vertical = np.array(vert, dtype=bool)
    t.n_gamma = n_gamma
    t.xline, t.yline = xline, yline
    t.leaf_width = width / n
    t.leaf_height = height / n
    t.n_boxes = nb
    t.leaves = [b for b in range(nb) if ca_l[b] < 0]
    return t


# ----------------------------------------------------------------------------------------------
# Leaf geometry and leaf stage (leafops.py:88-302, solver.py:184-247)
# ----------------------------------------------------------------------------------------------
class Geometry:
    """Restatement of LeafGeometry (leafops.py:88-214)."""

    def __init__(self, p, width, height):
        self.p = p
        self.cheb_x = cheb_nodes(p, (0.0, width))
        self.cheb_y = cheb_nodes(p, (0.0, height))
        self.gauss_x = (gauss_nodes(p) + 1.0) * 0.5 * width
        self.gauss_y = (gauss_nodes(p) + 1.0) * 0.5 * height
        Dx = cheb_diff_matrix(p, (0.0, width))
        Dy = cheb_diff_matrix(p, (0.0, height))
        I = np.eye(p)
        self.Dx, self.Dy = Dx, Dy
        # x1-major tensor grid: node (i, j) -> i*p + j (leafops.py:111-121)
        self.D1 = np.kron(Dx, I)
        self.D2 = np.kron(I, Dy)
        self.D1sq = np.kron(Dx @ Dx, I)
        self.D12 = np.kron(Dx, Dy)
        self.D2sq = np.kron(I, Dy @ Dy)
        self.grid_x = np.repeat(self.cheb_x, p)
        self.grid_y = np.tile(self.cheb_y, p)
        ii = np.arange(1, p - 1)
        self.J_i = (ii[:, None] * p + ii[None, :]).reshape(-1).astype(np.intp)
        r = np.arange(p - 1)
        # S owns SW, E owns SE, N owns NE, W owns NW (leafops.py:122-128)
        self.J_e = np.concatenate([r * p, (p - 1) * p + r, (r + 1) * p + (p - 1), r + 1]).astype(np.intp)
        self.L1 = self._l1()
        Qx = interp_matrix(self.cheb_x, self.gauss_x)
        Qy = interp_matrix(self.cheb_y, self.gauss_y)
        self.Qx, self.Qy = Qx, Qy
        self.L4 = np.zeros((4 * p, 4 * p))
        for s, Q in enumerate((Qx, Qy, Qx, Qy)):  # leafops.py:191-198
            self.L4[s * p:(s + 1) * p, s * p:(s + 1) * p] = Q
        g = lambda i, j: i * p + j
        L3 = np.array([self.D2[g(i, 0)] for i in range(p)] + [self.D1[g(p - 1, j)] for j in range(p)]
                      + [self.D2[g(i, p - 1)] for i in range(p)] + [self.D1[g(0, j)] for j in range(p)])
        self.L43 = self.L4 @ L3  # leafops.py:132, 181-189

    def _l1(self):
        """Gauss -> boundary-Chebyshev map with averaged corners (leafops.py:143-179)."""
        p = self.p
        PS = interp_matrix(self.gauss_x, self.cheb_x)
        PE = interp_matrix(self.gauss_y, self.cheb_y)
        S, E, N, W = (slice(k * p, (k + 1) * p) for k in range(4))
        L1 = np.zeros((4 * (p - 1), 4 * p))
        for i in range(p - 1):  # south (row 0 = SW corner)
            if i == 0:
                L1[i, S] = 0.5 * PS[0]
                L1[i, W] = 0.5 * PE[0]
            else:
                L1[i, S] = PS[i]
        o = p - 1
        for j in range(p - 1):  # east (row 0 = SE corner)
            if j == 0:
                L1[o + j, E] = 0.5 * PE[0]
                L1[o + j, S] = 0.5 * PS[p - 1]
            else:
                L1[o + j, E] = PE[j]
        o = 2 * (p - 1)
        for k, i in enumerate(range(1, p)):  # north (last = NE corner)
            if i == p - 1:
                L1[o + k, N] = 0.5 * PS[p - 1]
                L1[o + k, E] = 0.5 * PE[p - 1]
            else:
                L1[o + k, N] = PS[i]
        o = 3 * (p - 1)
        for k, j in enumerate(range(1, p)):  # west (last = NW corner)
            if j == p - 1:
                L1[o + k, W] = 0.5 * PE[p - 1]
                L1[o + k, N] = 0.5 * PS[0]
            else:
                L1[o + k, W] = PE[j]
        return L1


def assemble_operator(geom, vals):
    """Collocated operator A = -c11 D1sq - 2 c12 D12 - c22 D2sq + c1 D1 + c2 D2 + diag(c)
    (leafops.py:217-233). Scalar zero coefficients contribute nothing; the rest row-scale."""
    n = geom.p ** 2
    A = np.zeros((n, n))
    for key, M in (("c11", -geom.D1sq), ("c12", -2.0 * geom.D12), ("c22", -geom.D2sq),
                   ("c1", geom.D1), ("c2", geom.D2)):
        v = vals[key]
        if np.isscalar(v):
            if v != 0.0:
                A += v * M
        else:
            A += v[:, None] * M
    A[np.arange(n), np.arange(n)] += vals["c"]
    return A


def sample_coefficients(coeffs, tree, geom):
    """Sample the six coefficient fields on all leaf Chebyshev grids (solver.py:196-206)."""
    leaves = tree.leaves
    xlo = np.array([tree.xline[tree.cells[b][0]] for b in leaves])
    ylo = np.array([tree.yline[tree.cells[b][1]] for b in leaves])
    xs = xlo[:, None] + geom.grid_x[None, :]
    ys = ylo[:, None] + geom.grid_y[None, :]
    out = {}
    for name in COEFF_NAMES:
        f = coeffs[name]
        out[name] = f(xs, ys) if callable(f) else float(f)
        v = np.atleast_1d(out[name])
        if not np.all(np.isfinite(v)):
            bad = np.argwhere(~np.isfinite(np.broadcast_to(out[name], xs.shape)))
            i, k = bad[0] if bad.size else (0, 0)
            raise ValueError(f"coefficient {name} is not finite at node ({xs[i, k]}, {ys[i, k]})")
    return out


def group_leaves(fields, n_leaf):
    """Bitwise-identical coefficient samples share one group (solver.py:208-222).

    Returns (rep_leaf_positions in first-occurrence order, group_of_leaf)."""
    groups = OrderedDict()
    gid = np.empty(n_leaf, dtype=np.int64)
    for i in range(n_leaf):
        key = tuple(fields[nm] if np.isscalar(fields[nm]) else fields[nm][i].tobytes() for nm in COEFF_NAMES)
        g = groups.get(key)
        if g is None:
            g = len(groups)
            groups[key] = (g, i)
        else:
            g = g[0]
        gid[i] = g
    reps = np.array([v[1] for v in groups.values()], dtype=np.int64)
    return reps, gid


def leaf_operators(geom, fields, reps):
    """Psi, T and probe-condition estimates for each group representative (leafops.py:273-302,
    solver.py:226-246). Returns (Psi[n,196,60], T[n,64,64], cond[n])."""
    p2 = geom.p ** 2
    ng = len(reps)
    ni = geom.J_i.size
    probe = np.random.default_rng(1234).standard_normal((ni, 1))  # leafops.py:285-286
    Psi = np.empty((ng, ni, geom.J_e.size))
    T = np.empty((ng, 4 * geom.p, 4 * geom.p))
    cond = np.empty(ng)
    chunk = max(1, int(2e8 / (8 * p2 * p2)))  # solver.py:226
    for lo in range(0, ng, chunk):
        part = reps[lo:lo + chunk]
        A = np.empty((len(part), p2, p2))
        for j, i in enumerate(part):
            A[j] = assemble_operator(geom, {k: (v if np.isscalar(v) else v[i]) for k, v in fields.items()})
        Aii = A[:, geom.J_i][:, :, geom.J_i]
        Aie = A[:, geom.J_i][:, :, geom.J_e]
        rhs = np.concatenate([Aie, np.broadcast_to(probe, (len(part), ni, 1))], axis=2)
        sol = np.linalg.solve(Aii, rhs)  # LAPACK gesv, leafops.py:290
        anorm = np.abs(Aii).sum(axis=2).max(axis=1)
        cond[lo:lo + len(part)] = anorm * np.abs(sol[:, :, -1]).max(axis=1) / np.abs(probe).max()
        ps = -sol[:, :, :-1]
        Psi[lo:lo + len(part)] = ps
        L43L2 = geom.L43[:, geom.J_e][None] + geom.L43[:, geom.J_i] @ ps  # solver.py:241
        T[lo:lo + len(part)] = L43L2 @ geom.L1  # solver.py:242
    return Psi, T, cond


# ----------------------------------------------------------------------------------------------
# Merge (merge.py:68-119)
# ----------------------------------------------------------------------------------------------
def split_indices(Ie_a, Ie_b, I_i):
    """Positions of J1/J2/J3 in the child boundary lists (merge.py:68-89)."""
    pa = {int(v): k for k, v in enumerate(Ie_a)}
    pb = {int(v): k for k, v in enumerate(Ie_b)}
    j3a = np.array([pa[int(v)] for v in I_i], dtype=np.intp)
    j3b = np.array([pb[int(v)] for v in I_i], dtype=np.intp)
    ma = np.ones(len(Ie_a), bool)
    ma[j3a] = False
    mb = np.ones(len(Ie_b), bool)
    mb[j3b] = False
    return np.flatnonzero(ma), np.flatnonzero(mb), j3a, j3b


def merge_dtn(Ta, Tb, j1a, j2b, j3a, j3b):
    """S = (T33a - T33b)^{-1} [-T31a | T32b]; T = blkdiag(T11a, T22b) + [T13a; T23b] S
    (merge.py:92-119), via LAPACK getrf/getrs like the reference."""
    X = Ta[np.ix_(j3a, j3a)] - Tb[np.ix_(j3b, j3b)]
    R = np.concatenate([-Ta[np.ix_(j3a, j1a)], Tb[np.ix_(j3b, j2b)]], axis=1)
    lu = sla.lu_factor(X, check_finite=False)
    S = sla.lu_solve(lu, R, check_finite=False)
    if not np.all(np.isfinite(S)):
        raise FloatingPointError("non-finite solution operator")
    n1 = j1a.size
    T = np.zeros((n1 + j2b.size,) * 2)
    T[:n1, :n1] = Ta[np.ix_(j1a, j1a)]
    T[n1:, n1:] = Tb[np.ix_(j2b, j2b)]
    T += np.concatenate([Ta[np.ix_(j1a, j3a)], Tb[np.ix_(j2b, j3b)]]) @ S
    return S, T


# ----------------------------------------------------------------------------------------------
# Build / solve (solver.py:250-316) and null-mode-invariant extractors
# ----------------------------------------------------------------------------------------------
class OracleState:
    pass


def build(tree, coeffs, keep_T=False):
    """Dense bottom-up build (solver.py:250-289, switch_threshold=None branch).

    `coeffs` is a dict name -> scalar or callable(x, y). With keep_T=True every per-box T is
    retained in `state.T` (the reference frees children, solver.py:272-273).
    """
    geom = Geometry(tree.q, tree.leaf_width, tree.leaf_height)
    fields = sample_coefficients(coeffs, tree, geom)
    reps, gid = group_leaves(fields, len(tree.leaves))
    Psi, Tg, cond = leaf_operators(geom, fields, reps)
    bad = np.flatnonzero(cond > RESONANCE_COND)
    st = OracleState()
    st.tree, st.geom, st.reps, st.gid, st.cond = tree, geom, reps, gid, cond
    if bad.size:
        st.resonant_leaf = tree.leaves[int(reps[bad[0]])]
        raise ArithmeticError(f"leaf resonance at box {st.resonant_leaf}")
    st.psi_groups, st.T_groups = Psi, Tg
    store = {}
    for k, b in enumerate(tree.leaves):
        store[b] = Tg[gid[k]]
    st.S = {}
    st.T = {} if keep_T else None
    if keep_T:
        st.T.update(store)
    for b in range(tree.n_boxes - 1, -1, -1):
        a, c = tree.child_a[b], tree.child_b[b]
        if a < 0:
            continue
        j1a, j2b, j3a, j3b = split_indices(tree.I_e[a], tree.I_e[c], tree.I_i[b])
        S, T = merge_dtn(store.pop(a), store.pop(c), j1a, j2b, j3a, j3b)
        st.S[b] = S
        store[b] = T
        if keep_T:
            st.T[b] = T
    st.root_T = store[0]
    return st


def solve(st, f):
    """Top-down sweep u[I_i] = S u[I_e] (solver.py:303-316). `f` is (n_gamma,) or (n_gamma, b)."""
    tree = st.tree
    f = np.asarray(f, dtype=float)
    u = np.zeros((tree.points.shape[0],) + f.shape[1:])
    u[tree.I_e[0]] = f
    for b in range(tree.n_boxes):
        if tree.child_a[b] < 0:
            continue
        u[tree.I_i[b]] = st.S[b] @ u[tree.I_e[b]]
    return u


def leaf_cheb_boundary(st, u):
    """Per-leaf Chebyshev boundary values L1 u[I_e] (null-mode invariant).
    Returns (n_leaf, 4(p-1)[, b])."""
    tree, geom = st.tree, st.geom
    Ue = np.stack([u[tree.I_e[b]] for b in tree.leaves])
    return np.einsum("rc,lc...->lr...", geom.L1, Ue)


def leaf_flux(st, u):
    """Per-leaf flux T_leaf u[I_e] (null-mode invariant)."""
    tree = st.tree
    return np.stack([st.T_groups[st.gid[k]] @ u[tree.I_e[b]] for k, b in enumerate(tree.leaves)])


def leaf_cheb_field(st, u):
    """Full p x p Chebyshev field per leaf (solver.py:349-356), x1-major; invariant."""
    tree, geom = st.tree, st.geom
    we = leaf_cheb_boundary(st, u)
    out = np.zeros((len(tree.leaves), geom.p ** 2) + we.shape[2:])
    out[:, geom.J_e] = we
    out[:, geom.J_i] = np.einsum("lie,le...->li...", st.psi_groups[st.gid], we)
    return out


def unknowns(L, p):
    """BASELINE "unknowns" = 4^L p^2."""
    return (4 ** L) * p * p


def merge_flops(L, q):
    """Standard LAPACK count per depth: 2/3 n3^3 + 2 n3^2 ne + 2 n3 ne^2."""
    tot = 0.0
    for d in range(2 * L):
        n3, ne = depth_sizes(L, q, d)
        tot += (2 ** d) * (2.0 / 3.0 * n3 ** 3 + 2.0 * n3 ** 2 * ne + 2.0 * n3 * ne ** 2)
    return tot


def depth_sizes(L, q, d):
    """(n3, ne) of a parent at depth d (SURVEY.md §8 notation)."""
    j = d // 2
    if d % 2 == 0:
        side = 2 ** (L - j)
        return side * q, 4 * side * q
    w, h = 2 ** (L - j - 1), 2 ** (L - j)
    return w * q, 2 * (w + h) * q


def leaf_flops(p):
    ni, nb, ng = (p - 2) ** 2, 4 * (p - 1), 4 * p
    return 2.0 / 3.0 * ni ** 3 + 2.0 * ni ** 2 * (nb + 1) + 2.0 * ng * ni * nb + 2.0 * ng * nb * ng


def solve_flops(L, q, b):
    return 2.0 * b * sum((2 ** d) * depth_sizes(L, q, d)[0] * depth_sizes(L, q, d)[1] for d in range(2 * L))
