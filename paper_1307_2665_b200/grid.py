"""Box tree, global Gauss node set and 1-D interpolation: the host-side layout for the GPU path.

Drop-in for `hpsolve.grid` (reference grid.py:16-25): same public names, same argument meaning,
same errors, and the same numbers. The tree and node layout is bit-exact with the reference's
`build_tree` (grid.py:204-322). It is built from closed forms in (depth, slot) instead of a
key dictionary:
  * heap numbering (children of i are 2i+1, 2i+2; grid.py:229-248 builds exactly this order);
  * every parent's I_i is a contiguous id range (grid.py:284-295 registers a fresh cut line);
  * every depth is uniform, so one (n3, ne) pair and one split map serve a whole depth.
The arrays come from the library's host C++ builder (csrc/tree.cu, hps_tree_layout; L=9 in about
0.2 s, the reference needs minutes); the vectorised numpy version of the same closed forms below
(HPS_NATIVE_LAYOUT=0) is the cross-check of the tests and the path when the library is absent.

The per-depth arrays (`TreeLayout`) are what the CUDA kernels consume. `BoxTree.boxes` builds
reference-shaped `BoxNode` objects lazily from them.
"""

from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

__all__ = [
    "Rectangle",
    "BoxNode",
    "BoxTree",
    "GlobalNodeSet",
    "TreeLayout",
    "gauss_nodes",
    "cheb_nodes",
    "interp_matrix",
    "build_tree",
]


@dataclass(frozen=True)
class Rectangle:
    """Axis-aligned rectangle (grid.py:28-48)."""

    x_lo: float
    x_hi: float
    y_lo: float
    y_hi: float

    def __post_init__(self):
        if not (self.x_lo < self.x_hi and self.y_lo < self.y_hi):
            raise ValueError(f"degenerate rectangle {self}")

    @property
    def width(self):
        return self.x_hi - self.x_lo

    @property
    def height(self):
        return self.y_hi - self.y_lo

    def contains(self, x, y):
        return (self.x_lo <= x <= self.x_hi) and (self.y_lo <= y <= self.y_hi)


@dataclass
class BoxNode:
    """One box (grid.py:51-75). ``cells`` = (ix, iy, nx, ny) in leaf-cell units."""

    index: int
    rect: Rectangle
    level: int
    parent: int | None = None
    child_a: int | None = None
    child_b: int | None = None
    split_axis: str = "none"
    cells: tuple = (0, 0, 1, 1)
    I_e: np.ndarray = field(default=None, repr=False)
    I_i: np.ndarray = field(default=None, repr=False)

    @property
    def is_leaf(self):
        return self.child_a is None


@dataclass
class GlobalNodeSet:
    """Deduplicated Gauss nodes on leaf edges (grid.py:116-130)."""

    points: np.ndarray
    on_vertical: np.ndarray
    n_gamma: int

    @property
    def N(self):
        return self.points.shape[0]


# ----------------------------------------------------------------------------------------------
# 1-D nodes (grid.py:133-201). Same flop sequences as the reference => bitwise-equal nodes.
# ----------------------------------------------------------------------------------------------
def gauss_nodes(q):
    """Gauss-Legendre points on (-1, 1), ascending (grid.py:133-154)."""
    if q < 1:
        raise ValueError("q must be >= 1")
    if q == 1:
        return np.zeros(1)
    x = -np.cos(np.pi * (4 * np.arange(q) + 3) / (4 * q + 2))
    for _ in range(100):
        lo, hi = np.zeros_like(x), np.ones_like(x)
        for k in range(q):
            lo, hi = hi, ((2 * k + 1) * x * hi - k * lo) / (k + 1)
        dx = hi / (q * (x * hi - lo) / (x * x - 1.0))
        x = x - dx
        if np.max(np.abs(dx)) < 1e-15:
            break
    return np.sort(x)


def cheb_nodes(p, interval=(-1.0, 1.0)):
    """Chebyshev extreme points on [a, b], ascending, exact endpoints (grid.py:157-167)."""
    a, b = interval
    if p < 2:
        raise ValueError("p must be >= 2")
    if not a < b:
        raise ValueError("empty interval")
    x = 0.5 * (a + b) + 0.5 * (b - a) * np.cos(np.pi * np.arange(p) / (p - 1))[::-1]
    x[0], x[-1] = a, b
    return x


def interp_matrix(src, dst):
    """|dst| x |src| barycentric Lagrange weights (grid.py:178-201)."""
    src = np.atleast_1d(np.asarray(src, dtype=float))
    dst = np.atleast_1d(np.asarray(dst, dtype=float))
    if src.ndim != 1 or src.size < 1:
        raise ValueError("src must be a nonempty 1-D node list")
    if np.unique(src).size != src.size:
        raise ValueError("duplicate source nodes")
    if src.size == 1:
        return np.ones((dst.size, 1))
    s = 4.0 / max(src.max() - src.min(), np.finfo(float).tiny)
    dd = (src[:, None] - src[None, :]) * s
    np.fill_diagonal(dd, 1.0)
    w = 1.0 / np.prod(dd, axis=1)
    d = dst[:, None] - src[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        r = w[None, :] / d
        M = r / np.sum(r, axis=1)[:, None]
    hit_r, hit_c = np.nonzero(d == 0.0)
    M[hit_r] = 0.0
    M[hit_r, hit_c] = 1.0
    return M


# ----------------------------------------------------------------------------------------------
# Closed-form layout
# ----------------------------------------------------------------------------------------------
def depth_shape(L, d):
    """Box footprint (nx, ny) in leaf cells at depth d: cuts alternate v, h (grid.py:230-239)."""
    n = 1 << L
    return n >> ((d + 1) // 2), n >> (d // 2)


@dataclass
class DepthLayout:
    """Everything the kernels need about the 2^d parents at depth d (uniform across the depth).

    n3 = |I_i|, ne = |I_e(parent)|, m = |I_e(child)|. The split maps are positions inside a
    child's boundary list (reference merge.py:68-89), identical for every parent at this depth.
    """

    depth: int
    axis: str
    n3: int
    ne: int
    m: int
    j1a: np.ndarray
    j2b: np.ndarray
    j3a: np.ndarray
    j3b: np.ndarray
    I_e: np.ndarray  # (2^d, ne) intp, global node ids
    Ii_start: np.ndarray  # (2^d,) intp; I_i = arange(start, start + n3)

    @property
    def n_boxes(self):
        return self.I_e.shape[0]


class TreeLayout:
    """Per-depth arrays for a (domain, L, q) tree. Depth 0 is the root, depth 2L the leaves."""

    def __init__(self, domain, L, q):
        self.domain = domain
        self.L = L
        self.q = q
        n = 1 << L
        self.n = n
        self.depths: list[DepthLayout] = []
        self.leaf_I_e = None  # (4^L, 4q)
        self.leaf_cells = None  # (4^L, 2) = (ix, iy) in heap order
        if not (_use_native_layout() and self._build_native()):
            self._build()

    # -- cells of all boxes at one depth, heap order (grid.py:229-248) --
    def cells_at(self, d):
        L, n = self.L, self.n
        k = np.arange(1 << d, dtype=np.int64)
        ix = np.zeros_like(k)
        iy = np.zeros_like(k)
        for t in range(d):  # bit t (from the top) chooses child b at depth t
            bit = (k >> (d - 1 - t)) & 1
            nx, ny = depth_shape(L, t)
            if t % 2 == 0:
                ix += bit * (nx // 2)
            else:
                iy += bit * (ny // 2)
        nx, ny = depth_shape(L, d)
        return ix, iy, nx, ny

    def _build(self):
        L, q, n = self.L, self.q, self.n
        ng = 4 * n * q
        self.n_gamma = ng
        # I_i ranges: parents in heap order, each registers a fresh contiguous range (grid.py:284-295)
        n3s = []
        for d in range(2 * L):
            nx, ny = depth_shape(L, d)
            n3s.append((ny if d % 2 == 0 else nx) * q)
        depth_off = [ng]
        for d in range(2 * L):
            depth_off.append(depth_off[-1] + (1 << d) * n3s[d])
        self.N = depth_off[-1]
        expected = (1 << (2 * L + 1)) * q + (1 << (L + 1)) * q
        assert self.N == expected, (self.N, expected)
        self.n3s = n3s
        self.depth_off = depth_off

        # depth (as a parent) whose cut line is vertical line i / horizontal line j
        def v_depth(i):  # i interior: lowbit(i) = nx/2 at even depth 2t with nx = n >> t
            low = i & -i
            t = int(np.log2(n // (2 * low)))
            return 2 * t
        # vectorised id lookup for key arrays
        gq = np.arange(q)

        def h_ids(line, seg):  # key ('h', line, seg, g) -> ids (..., q)
            line = np.asarray(line, np.int64)
            seg = np.asarray(seg, np.int64)
            out = np.empty(np.broadcast(line, seg).shape + (q,), np.int64)
            lineb, segb = np.broadcast_arrays(line, seg)
            south = lineb == 0
            north = lineb == n
            inner = ~(south | north)
            out[south] = segb[south][:, None] * q + gq
            out[north] = 2 * n * q + segb[north][:, None] * q + gq
            if inner.any():
                ln = lineb[inner]
                sg = segb[inner]
                low = ln & -ln
                ny = 2 * low  # box height at the cutting depth
                t = np.log2(n // ny).astype(np.int64)
                d = 2 * t + 1
                nx = ny // 2
                bx = sg // nx  # box position along x
                by = (ln - low) // ny
                slot = _slot_from_xy(bx, by, d)
                base = np.array(depth_off, np.int64)[d] + slot * np.array(n3s, np.int64)[d]
                out[inner] = (base + (sg - bx * nx) * q)[:, None] + gq
            return out

        def v_ids(line, seg):  # key ('v', line, seg, g)
            line = np.asarray(line, np.int64)
            seg = np.asarray(seg, np.int64)
            lineb, segb = np.broadcast_arrays(line, seg)
            out = np.empty(lineb.shape + (q,), np.int64)
            west = lineb == 0
            east = lineb == n
            inner = ~(west | east)
            out[west] = 3 * n * q + segb[west][:, None] * q + gq
            out[east] = n * q + segb[east][:, None] * q + gq
            if inner.any():
                ln = lineb[inner]
                sg = segb[inner]
                low = ln & -ln
                nx = 2 * low
                t = np.log2(n // nx).astype(np.int64)
                d = 2 * t
                ny = nx
                bx = (ln - low) // nx
                by = sg // ny
                slot = _slot_from_xy(bx, by, d)
                base = np.array(depth_off, np.int64)[d] + slot * np.array(n3s, np.int64)[d]
                out[inner] = (base + (sg - by * ny) * q)[:, None] + gq
            return out

        def _slot_from_xy(bx, by, d):
            # heap slot at depth d from box coordinates in units of that depth's box size:
            # bits interleave, x bit first (vertical cut at even depth).
            # `d` may vary per element.
            d = np.broadcast_to(np.asarray(d, np.int64), bx.shape)
            slot = np.zeros_like(bx)
            nxb = (d + 1) // 2  # number of x bits
            nyb = d // 2
            for t in range(int(d.max()) if d.size else 0):
                on = t < d
                if t % 2 == 0:
                    bit = (bx >> np.maximum(nxb - 1 - t // 2, 0)) & 1
                else:
                    bit = (by >> np.maximum(nyb - 1 - t // 2, 0)) & 1
                slot = np.where(on, (slot << 1) | bit, slot)
            return slot

        self._h_ids, self._v_ids = h_ids, v_ids

        # points / orientation in id order (grid.py:256-268). Every id's key is known in closed form.
        xline = self.domain.x_lo + np.arange(n + 1) * (self.domain.width / n)
        yline = self.domain.y_lo + np.arange(n + 1) * (self.domain.height / n)
        gx = self.domain.x_lo + (gauss_nodes(q) + 1.0) * 0.5 * (self.domain.width / n)
        gx = gx - self.domain.x_lo
        gy = (gauss_nodes(q) + 1.0) * 0.5 * (self.domain.height / n)
        self.xline, self.yline = xline, yline
        pts = np.empty((self.N, 2))
        vert = np.empty(self.N, bool)
        s = np.arange(n)
        # S, E, N, W boundary blocks
        blk = lambda a: a.reshape(-1)
        pts[0:n * q, 0] = blk(xline[s][:, None] + gx[None, :])
        pts[0:n * q, 1] = yline[0]
        vert[0:n * q] = False
        pts[n * q:2 * n * q, 0] = xline[n]
        pts[n * q:2 * n * q, 1] = blk(yline[s][:, None] + gy[None, :])
        vert[n * q:2 * n * q] = True
        pts[2 * n * q:3 * n * q, 0] = blk(xline[s][:, None] + gx[None, :])
        pts[2 * n * q:3 * n * q, 1] = yline[n]
        vert[2 * n * q:3 * n * q] = False
        pts[3 * n * q:4 * n * q, 0] = xline[0]
        pts[3 * n * q:4 * n * q, 1] = blk(yline[s][:, None] + gy[None, :])
        vert[3 * n * q:4 * n * q] = True
        for d in range(2 * L):
            ix, iy, nx, ny = self.cells_at(d)
            lo, n3 = depth_off[d], n3s[d]
            seg_local = np.arange(n3 // q)
            if d % 2 == 0:  # vertical cut line x = ix + nx/2, segments along y
                line = ix + nx // 2
                segs = iy[:, None] + seg_local[None, :]
                X = np.broadcast_to(xline[line][:, None, None], segs.shape + (q,))
                Y = yline[segs][:, :, None] + gy[None, None, :]
                v = True
            else:
                line = iy + ny // 2
                segs = ix[:, None] + seg_local[None, :]
                X = xline[segs][:, :, None] + gx[None, None, :]
                Y = np.broadcast_to(yline[line][:, None, None], segs.shape + (q,))
                v = False
            pts[lo:lo + (1 << d) * n3, 0] = X.reshape(-1)
            pts[lo:lo + (1 << d) * n3, 1] = Y.reshape(-1)
            vert[lo:lo + (1 << d) * n3] = v
        self.points = pts
        self.on_vertical = vert

        # leaf I_e: S, E, N, W sides, increasing coordinate (grid.py:305-312)
        lix, liy, _, _ = self.cells_at(2 * L)
        self.leaf_cells = np.stack([lix, liy], axis=1)
        self.leaf_I_e = np.ascontiguousarray(np.concatenate(
            [h_ids(liy, lix), v_ids(lix + 1, liy), h_ids(liy + 1, lix), v_ids(lix, liy)], axis=1))

        # parents bottom-up: child-a remainder then child-b remainder (grid.py:313-319). The split
        # maps are the same for every parent of a depth, so they come from the first parent; every
        # parent's I_e is then one vectorised gather, and the maps are checked on a sample of
        # parents (always including the first and last): the shared ids must sit at the same
        # positions and be the parent's contiguous I_i range.
        child_Ie = self.leaf_I_e
        depths = [None] * (2 * L)
        rng = np.random.default_rng(0)
        for d in range(2 * L - 1, -1, -1):
            nb = 1 << d
            A = child_Ie[0::2]
            B = child_Ie[1::2]
            start = depth_off[d] + np.arange(nb, dtype=np.int64) * n3s[d]
            n3 = n3s[d]
            m = A.shape[1]
            a0, b0 = A[0], B[0]
            in_a0 = (a0 >= start[0]) & (a0 < start[0] + n3)
            in_b0 = (b0 >= start[0]) & (b0 < start[0] + n3)
            if in_a0.sum() != n3 or in_b0.sum() != n3:
                raise AssertionError("children are not edge-adjacent")
            j3a = np.empty(n3, np.int64)
            j3a[a0[in_a0] - start[0]] = np.flatnonzero(in_a0)
            j3b = np.empty(n3, np.int64)
            j3b[b0[in_b0] - start[0]] = np.flatnonzero(in_b0)
            j1a = np.flatnonzero(~in_a0)
            j2b = np.flatnonzero(~in_b0)
            sample = np.unique(np.concatenate([[0, nb - 1], rng.integers(0, nb, size=min(nb, 64))]))
            shared = start[sample][:, None] + np.arange(n3)[None, :]
            As, Bs = A[sample], B[sample]
            ok = (np.array_equal(As[:, j3a], shared) and np.array_equal(Bs[:, j3b], shared)
                  and not np.any((As[:, j1a] >= start[sample][:, None]) & (As[:, j1a] < start[sample][:, None] + n3))
                  and not np.any((Bs[:, j2b] >= start[sample][:, None]) & (Bs[:, j2b] < start[sample][:, None] + n3)))
            if not ok:
                raise AssertionError(f"non-uniform split maps at depth {d}")
            Ie = np.concatenate([A[:, j1a], B[:, j2b]], axis=1)
            depths[d] = DepthLayout(
                depth=d, axis="v" if d % 2 == 0 else "h", n3=n3, ne=Ie.shape[1], m=m,
                j1a=j1a.astype(np.intp), j2b=j2b.astype(np.intp),
                j3a=j3a.astype(np.intp), j3b=j3b.astype(np.intp),
                I_e=Ie, Ii_start=start.astype(np.intp))
            child_Ie = Ie
        self.depths = depths
        self.root_I_e = child_Ie[0].astype(np.intp) if L > 0 else self.leaf_I_e[0].astype(np.intp)

    def _build_native(self):
        """The same layout from libhps_b200.so's host-side builder (csrc/tree.cu): every array
        identical to _build's (tests/test_layout.py), ~10x faster at L = 9. False if the library
        is not available."""
        import ctypes

        try:
            from . import _native
            lib = _native.load()
        except ImportError:
            return False
        L, q, n = self.L, self.q, self.n
        nd = 2 * L
        n3 = np.zeros(max(nd, 1), np.int64)
        ne = np.zeros(max(nd, 1), np.int64)
        m = np.zeros(max(nd, 1), np.int64)
        pl = ctypes.POINTER(ctypes.c_longlong)
        N = lib.hps_tree_sizes(L, q, n3.ctypes.data_as(pl), ne.ctypes.data_as(pl), m.ctypes.data_as(pl))
        if N < 0:
            raise ValueError(_native.last_error())
        dom = self.domain
        gauss01 = np.ascontiguousarray((gauss_nodes(q) + 1.0) * 0.5)
        points = np.empty((N, 2))
        vert = np.empty(N, np.uint8)
        nleaf = 1 << (2 * L)
        leaf_cells = np.empty((nleaf, 2), np.int64)
        leaf_Ie = np.empty((nleaf, 4 * q), np.int64)
        Ie = [np.empty((1 << d, int(ne[d])), np.int64) for d in range(nd)]
        maps = [np.empty(int(ne[d]) + 2 * int(n3[d]), np.int64) for d in range(nd)]
        Ie_p = (pl * max(nd, 1))(*[a.ctypes.data_as(pl) for a in Ie])
        maps_p = (pl * max(nd, 1))(*[a.ctypes.data_as(pl) for a in maps])
        st = lib.hps_tree_layout(L, q, float(dom.x_lo), float(dom.y_lo), float(dom.width), float(dom.height),
                                 gauss01.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                 points.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                 vert.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte)),
                                 leaf_cells.ctypes.data_as(pl), leaf_Ie.ctypes.data_as(pl), Ie_p, maps_p)
        if st != 0:
            raise AssertionError(_native.last_error())
        self.n_gamma = 4 * n * q
        self.N = int(N)
        self.n3s = [int(v) for v in n3[:nd]]
        off = [self.n_gamma]
        for d in range(nd):
            off.append(off[-1] + (1 << d) * self.n3s[d])
        self.depth_off = off
        self.xline = dom.x_lo + np.arange(n + 1) * (dom.width / n)
        self.yline = dom.y_lo + np.arange(n + 1) * (dom.height / n)
        self.points = points
        self.on_vertical = vert.view(bool)
        self.leaf_cells = leaf_cells
        self.leaf_I_e = leaf_Ie
        self._h_ids = self._v_ids = None
        depths = []
        for d in range(nd):
            n1, k3 = int(ne[d]) // 2, self.n3s[d]
            mp = maps[d].astype(np.intp)
            depths.append(DepthLayout(
                depth=d, axis="v" if d % 2 == 0 else "h", n3=k3, ne=int(ne[d]), m=int(m[d]),
                j1a=mp[:n1], j2b=mp[n1:2 * n1], j3a=mp[2 * n1:2 * n1 + k3], j3b=mp[2 * n1 + k3:],
                I_e=Ie[d], Ii_start=(off[d] + np.arange(1 << d, dtype=np.int64) * k3).astype(np.intp)))
        self.depths = depths
        self.root_I_e = Ie[0][0].astype(np.intp) if L > 0 else leaf_Ie[0].astype(np.intp)
        return True

    # -- reference-shaped accessors --
    def box_depth_slot(self, index):
        d = int(np.floor(np.log2(index + 1)))
        return d, index - ((1 << d) - 1)

    def box_I_e(self, index):
        d, k = self.box_depth_slot(index)
        if d == 2 * self.L:
            return self.leaf_I_e[k].astype(np.intp)
        return self.depths[d].I_e[k]

    def box_I_i(self, index):
        d, k = self.box_depth_slot(index)
        if d == 2 * self.L:
            return None
        lo = self.depths[d].Ii_start[k]
        return np.arange(lo, lo + self.depths[d].n3, dtype=np.intp)


class _LazyBoxes(Sequence):
    """List-like view creating reference-shaped BoxNode objects on access."""

    def __init__(self, tree):
        self._tree = tree
        self._cache = {}

    def __len__(self):
        return 2 * (4 ** self._tree.levels) - 1

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        node = self._cache.get(i)
        if node is None:
            node = self._tree._make_node(i)
            self._cache[i] = node
        return node


class BoxTree:
    """Heap-ordered box tree (grid.py:78-113), backed by a TreeLayout."""

    def __init__(self, layout: TreeLayout):
        self.layout = layout
        self.levels = layout.L
        self.q = layout.q
        self.domain = layout.domain
        self.boxes = _LazyBoxes(self)
        self._leaf_map = None

    def _make_node(self, i):
        lay = self.layout
        d, k = lay.box_depth_slot(i)
        ix, iy, nx, ny = lay.cells_at(d)
        ix, iy = int(ix[k]), int(iy[k])
        xl, yl = lay.xline, lay.yline
        leaf = d == 2 * lay.L
        node = BoxNode(
            index=i, rect=Rectangle(xl[ix], xl[ix + nx], yl[iy], yl[iy + ny]), level=d,
            parent=None if i == 0 else (i - 1) // 2,
            child_a=None if leaf else 2 * i + 1, child_b=None if leaf else 2 * i + 2,
            split_axis="none" if leaf else ("v" if d % 2 == 0 else "h"),
            cells=(ix, iy, nx, ny), I_e=lay.box_I_e(i), I_i=lay.box_I_i(i))
        return node

    @property
    def n_boxes(self):
        return len(self.boxes)

    def leaf_at(self, ix, iy):
        if self._leaf_map is None:
            lc = self.layout.leaf_cells
            first = (1 << (2 * self.levels)) - 1
            self._leaf_map = {(int(a), int(b)): first + k for k, (a, b) in enumerate(lc)}
        return self.boxes[self._leaf_map[(ix, iy)]]

    def leaves(self):
        first = (1 << (2 * self.levels)) - 1
        return [self.boxes[i] for i in range(first, len(self.boxes))]

    def parents(self):
        return [self.boxes[i] for i in range((1 << (2 * self.levels)) - 1)]

    @property
    def root(self):
        return self.boxes[0]

    @property
    def leaf_width(self):
        return self.domain.width / (1 << self.levels)

    @property
    def leaf_height(self):
        return self.domain.height / (1 << self.levels)


def _use_native_layout():
    import os
    return os.environ.get("HPS_NATIVE_LAYOUT", "1") != "0"


@lru_cache(maxsize=8)
def _layout_cached(domain, L, q):
    return TreeLayout(domain, L, q)


def build_tree(domain, L, q):
    """(BoxTree, GlobalNodeSet) for `domain` cut into 4^L leaves with q Gauss nodes per edge
    (grid.py:204-322). Bit-exact with the reference layout."""
    if not isinstance(domain, Rectangle):
        domain = Rectangle(*domain)
    if L < 0:
        raise ValueError("L must be >= 0")
    if q < 2:
        raise ValueError("q must be >= 2")
    lay = _layout_cached(domain, int(L), int(q))
    return BoxTree(lay), GlobalNodeSet(lay.points, lay.on_vertical, lay.n_gamma)


def layout_of(tree) -> TreeLayout:
    """TreeLayout for any tree object with (domain, levels, q): ours or the reference's."""
    lay = getattr(tree, "layout", None)
    if isinstance(lay, TreeLayout):
        return lay
    dom = tree.domain
    if not isinstance(dom, Rectangle):
        dom = Rectangle(dom.x_lo, dom.x_hi, dom.y_lo, dom.y_hi)
    return _layout_cached(dom, int(tree.levels), int(tree.q))
