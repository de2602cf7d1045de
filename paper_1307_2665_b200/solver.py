"""Build and solve stages on B200: drop-in for `hpsolve.solver` (reference solver.py:40-50).

Host code only. It samples coefficients, groups leaves, owns device memory (through torch) and
enqueues the C-ABI calls: one leaf-stage call, one merge call per depth, one solve call per depth.
All arithmetic runs in libhps_b200.so. The returned `SolverState` has the reference's
attributes. The device-resident operators (`S`, `psi`, `root_T`) are copied to numpy only when
accessed.

Differences from the reference, all documented in DESIGN.md:
  * `eps`, `switch_threshold` and `hbs_leaf_size` are accepted and ignored. The GPU path is
    dense by design; the reference's HBS branch is out of scope.
  * The interface systems are deflated along their analytic corner null modes, so `S` is the
    unique gauge-fixed solution (V^T S = 0) instead of the reference's rounding-dependent one.
    T, and every null-mode-invariant function of u, match the reference.
  * `solve` also accepts a batch F of shape (|Gamma|, b) and returns (N, b).
"""

from __future__ import annotations

import ctypes
import math
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np

from . import _native, instrumentation
from .errors import LeafResonanceError, MergeResonanceError
from .grid import interp_matrix, layout_of
from .leafops import RESONANCE_COND, LeafGeometry

__all__ = [
    "DtnOperator",
    "SolutionOperator",
    "SolverState",
    "build",
    "prepare",
    "build_device",
    "check_build",
    "solve",
    "solve_device",
    "apply_global_dtn",
    "post_process",
    "boundary_flux_at",
    "leaf_fields",
    "gauge_fixed_solution",
    "Pipeline",
    "BuildGraph",
    "memory_report",
]

COEFF_NAMES = ("c11", "c12", "c22", "c1", "c2", "c")
ctypes_vp = ctypes.c_void_p
ctypes_d = ctypes.c_double


def _torch():
    import torch

    return torch


def _device_apply(A, x):
    """A @ x for a device matrix A (m x k) and host x (k,) or (k, b), on the device (the library's
    DGEMM): the operator containers never compute on the host."""
    torch = _torch()
    xv = np.asarray(x, dtype=float)
    single = xv.ndim == 1
    X = xv[:, None] if single else xv
    m, k = A.shape
    if X.shape[0] != k:
        raise ValueError(f"operand has {X.shape[0]} rows, the operator {k} columns")
    b = X.shape[1]
    ld = -(-b // 2) * 2
    Xd = torch.zeros((k, ld), dtype=torch.float64, device=A.device)
    Xd[:, :b] = torch.from_numpy(np.ascontiguousarray(X)).to(A.device)
    out = torch.empty((m, ld), dtype=torch.float64, device=A.device)
    Ac = A.contiguous()
    with torch.cuda.device(A.device):
        _native.check(_native.load().hps_dgemm_batched(
            _native.context(), m, ld, k, 1, 1.0, _native.ptr(Ac), k, 0, _native.ptr(Xd), ld, 0, None, 0, 0.0,
            _native.ptr(out), ld, 0, _native.stream_ptr()), "hps_dgemm_batched")
    r = out[:, :b].cpu().numpy()
    return r[:, 0].copy() if single else r


# ----------------------------------------------------------------------------------------------
# Reference-shaped operator containers (solver.py:53-119), backed by device tensors
# ----------------------------------------------------------------------------------------------
class DtnOperator:
    """A box DtN map (solver.py:53-77). `dense` materialises the device tensor to numpy."""

    def __init__(self, dense=None, hbs=None, device_tensor=None):
        if hbs is not None:
            raise ValueError("the B200 path is dense-only (HBS is out of scope)")
        if (dense is None) == (device_tensor is None):
            raise ValueError("exactly one of dense/device_tensor required")
        self._host = dense
        self.device_tensor = device_tensor
        self.hbs = None

    @property
    def dense(self):
        if self._host is None:
            self._host = self.device_tensor.cpu().numpy()
        return self._host

    @property
    def is_dense(self):
        return True

    @property
    def dim(self):
        t = self.device_tensor if self.device_tensor is not None else self._host
        return t.shape[0]

    def apply(self, x):
        return _device_apply(self.device_tensor, x) if self.device_tensor is not None else self._host @ x

    def to_dense(self):
        return self.dense

    def n_stored_entries(self):
        t = self.device_tensor if self.device_tensor is not None else self._host
        return int(np.prod(t.shape))


class SolutionOperator:
    """Parent map u_e -> u_i (solver.py:80-102), a view into the per-depth device S tensor."""

    def __init__(self, dense=None, factors=None, device_tensor=None):
        if factors is not None:
            raise ValueError("the B200 path is dense-only (low-rank factors are out of scope)")
        self._host = dense
        self.device_tensor = device_tensor
        self.factors = None

    @property
    def dense(self):
        if self._host is None:
            self._host = self.device_tensor.cpu().numpy()
        return self._host

    @property
    def is_dense(self):
        return True

    def apply(self, u_e):
        return _device_apply(self.device_tensor, u_e) if self.device_tensor is not None else self._host @ u_e

    def n_stored_entries(self):
        t = self.device_tensor if self.device_tensor is not None else self._host
        return int(np.prod(t.shape))


class _LazyS(Mapping):
    """parent box index -> SolutionOperator over the per-depth S tensors."""

    def __init__(self, S_levels, L):
        self._S = S_levels
        self._n = (1 << (2 * L)) - 1

    def __getitem__(self, idx):
        if not 0 <= idx < self._n:
            raise KeyError(idx)
        d = int(math.floor(math.log2(idx + 1)))
        return SolutionOperator(device_tensor=self._S[d][idx - ((1 << d) - 1)])

    def __iter__(self):
        return iter(range(self._n))

    def __len__(self):
        return self._n


class _LazyPsi(Mapping):
    """leaf box index -> Psi (numpy); leaves of one coefficient group share one array object."""

    def __init__(self, psi_groups, leaf_group, first_leaf):
        self._dev = psi_groups
        self._gid = leaf_group
        self._first = first_leaf
        self._host = {}

    def group_array(self, g):
        a = self._host.get(g)
        if a is None:
            a = self._dev[g].cpu().numpy()
            self._host[g] = a
        return a

    def __getitem__(self, idx):
        k = idx - self._first
        if not 0 <= k < self._gid.size:
            raise KeyError(idx)
        return self.group_array(int(self._gid[k]))

    def __iter__(self):
        return iter(range(self._first, self._first + self._gid.size))

    def __len__(self):
        return int(self._gid.size)


@dataclass
class SolverState:
    """All built operators (solver.py:105-119) plus the device-resident level tensors."""

    tree: object
    nodes: object
    coeffs: object
    q: int
    eps: float
    switch_threshold: float
    hbs_leaf_size: int
    geometry: LeafGeometry
    psi: Mapping
    S: Mapping
    root_T: DtnOperator
    rank_stats: dict = field(default_factory=dict)
    n_leaf_groups: int = 0
    # device side
    layout: object = None
    S_levels: list = None
    Ie_levels: list = None
    psi_groups: object = None
    T_leaf_groups: object = None
    leaf_group: np.ndarray = None
    root_Ie_dev: object = None
    device: object = None
    level_T: list = None  # per-depth T tensors when build(..., keep_level_T=True)


# ----------------------------------------------------------------------------------------------
# Build
# ----------------------------------------------------------------------------------------------
_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        import concurrent.futures
        import os

        _POOL = concurrent.futures.ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1)))
    return _POOL


def _eval_field(f, xs, ys, threads=True, out=None):
    """f(xs, ys) for a pointwise coefficient callable. Large evaluations run on leaf-aligned row
    chunks in a thread pool (numpy ufuncs release the GIL). Each element is computed by the same
    SIMD code path as in a single call, since chunks are whole leaves, 256 points each.
    `out(shape)` optionally allocates the result (e.g. in pinned host memory); the chunks are then
    written straight into it instead of being concatenated. Returns (values, all_finite): the
    finiteness check runs per chunk inside the workers."""
    n = xs.shape[0]
    if not threads or n < 256:
        v = f(xs, ys)
        return v, bool(np.all(np.isfinite(v)))
    nchunk = max(1, min(16, n // 64))
    bounds = np.linspace(0, n, nchunk + 1).astype(int)
    first = f(xs[bounds[0]:bounds[1]], ys[bounds[0]:bounds[1]])
    if np.isscalar(first) or np.ndim(first) == 0:  # the callable returned a scalar
        v = f(xs, ys)
        return v, bool(np.all(np.isfinite(v)))
    res = out(xs.shape) if out is not None else np.empty(xs.shape)
    res[bounds[0]:bounds[1]] = np.broadcast_to(np.asarray(first, dtype=float), (bounds[1] - bounds[0], xs.shape[1]))
    ok0 = bool(np.all(np.isfinite(res[bounds[0]:bounds[1]])))

    def run(ab):
        b0, b1 = ab
        q = f(xs[b0:b1], ys[b0:b1])
        if np.isscalar(q) or np.ndim(q) == 0:
            return None
        res[b0:b1] = np.broadcast_to(np.asarray(q, dtype=float), (b1 - b0, xs.shape[1]))
        return bool(np.all(np.isfinite(res[b0:b1])))

    flags = list(_pool().map(run, zip(bounds[1:-1], bounds[2:])))
    if any(fl is None for fl in flags):
        v = f(xs, ys)
        return v, bool(np.all(np.isfinite(v)))
    return res, ok0 and all(flags)


_POINTS = {}


def _leaf_points(lay, geom):
    """Chebyshev grid points of every leaf (heap leaf order), cached per (tree, geometry)."""
    key = (id(lay), geom.p, geom.width, geom.height)
    v = _POINTS.get(key)
    if v is None:
        lc = lay.leaf_cells
        xs = lay.xline[lc[:, 0]][:, None] + geom.grid_x[None, :]
        ys = lay.yline[lc[:, 1]][:, None] + geom.grid_y[None, :]
        xs.setflags(write=False)
        ys.setflags(write=False)
        v = _POINTS[key] = (xs, ys)
    return v


def _sample(coeffs, lay, geom, threads=True, out=None):
    """Coefficient samples on all leaf Chebyshev grids, heap leaf order (solver.py:196-206)."""
    xs, ys = _leaf_points(lay, geom)
    fields = {}
    for name in COEFF_NAMES:
        f = getattr(coeffs, name)
        if callable(f):
            fields[name], finite = _eval_field(f, xs, ys, threads, out)
        else:
            fields[name] = float(f)
            finite = bool(np.isfinite(fields[name]))
        if not finite:
            bad = np.argwhere(~np.isfinite(np.broadcast_to(fields[name], xs.shape)))
            i, k = (bad[0] if bad.size else (0, 0))
            raise ValueError(f"coefficient {name} is not finite at node ({xs[i, k]}, {ys[i, k]})")
        if not np.isscalar(fields[name]):
            fields[name] = np.ascontiguousarray(np.broadcast_to(np.asarray(fields[name], dtype=float), xs.shape))
    return fields


def _group(fields, n_leaf):
    """Group leaves whose six sample rows are bitwise equal (solver.py:208-222).

    Returns (rep leaf positions in first-occurrence order, group id per leaf). Exact: rows are
    bucketed by a 64-bit hash of their bit patterns, then every row is compared bitwise with its
    bucket's first row. A hash collision (never observed) falls back to exact byte-key sorting.
    """
    arrays = [np.ascontiguousarray(fields[n]).view(np.uint64).reshape(n_leaf, -1)
              for n in COEFF_NAMES if not np.isscalar(fields[n])]
    if not arrays:
        return np.zeros(1, np.int64), np.zeros(n_leaf, np.int64)
    rng = np.random.default_rng(0x5eed)
    h = np.zeros(n_leaf, np.uint64)
    with np.errstate(over="ignore"):
        for a in arrays:  # wrapping 64-bit dot products of the bit patterns
            h += a @ (rng.integers(1, 2 ** 63, size=a.shape[1], dtype=np.uint64) | np.uint64(1))
    _, first, inv = np.unique(h, return_index=True, return_inverse=True)
    inv = inv.reshape(-1)
    rep_of = first[inv]
    if not all(np.array_equal(a, a[rep_of]) for a in arrays):  # collision: exact fallback
        rows = np.concatenate(arrays, axis=1)
        key = rows.view(np.uint8).view(np.dtype((np.void, rows.shape[1] * 8))).reshape(n_leaf)
        _, first, inv = np.unique(key, return_index=True, return_inverse=True)
        inv = inv.reshape(-1)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    return first[order].astype(np.int64), rank[inv].astype(np.int64)


def _group_device(dev_fields, n_leaf):
    """_group on the device (solver.py:208-222): hash every leaf's sample rows (hps_leaf_hash),
    bucket by hash, then check every leaf bitwise against its bucket's first leaf (hps_leaf_verify).
    Returns (reps, gid) as device int64 tensors in _group's order (groups by first occurrence), or
    None if the bitwise check found a hash collision (the caller regroups exactly on the host)."""
    torch = _torch()
    lib = _native.load()
    dev = dev_fields[0].device
    row = int(dev_fields[0].shape[1])
    stream = _native.stream_ptr()
    ptrs = (ctypes_vp * len(dev_fields))(*[_native.ptr(t).value for t in dev_fields])
    h = torch.empty(n_leaf, dtype=torch.int64, device=dev)
    _native.check(lib.hps_leaf_hash(n_leaf, row, len(dev_fields), ptrs, _native.ptr(h), stream), "hps_leaf_hash")
    _, inv = torch.unique(h, sorted=True, return_inverse=True)
    ng = int(inv.max()) + 1
    ar = torch.arange(n_leaf, device=dev)
    first = torch.full((ng,), n_leaf, dtype=torch.int64, device=dev).scatter_reduce_(0, inv, ar, "amin")
    rep_of = first[inv].contiguous()
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.check(lib.hps_leaf_verify(n_leaf, row, len(dev_fields), ptrs, _native.ptr(rep_of), _native.ptr(bad),
                                      stream), "hps_leaf_verify")
    order = torch.argsort(first)
    rank = torch.empty_like(order)
    rank[order] = torch.arange(ng, device=dev)
    if int(bad.item()):
        return None
    return first[order], rank[inv]


class _DeviceLayout:
    """Per-(tree, device) int32 tables: merge split maps, corner-mode vectors, I_e gathers."""

    _cache = {}

    @classmethod
    def get(cls, lay, geom, device):
        key = (id(lay), geom.p, geom.width, geom.height, str(device))
        v = cls._cache.get(key)
        if v is None:
            v = cls(lay, geom, device)
            cls._cache[key] = v
        return v

    def __init__(self, lay, geom, device):
        torch = _torch()
        self.maps, self.vmode, self.Ie = [], [], []
        for dl in lay.depths:
            m = np.concatenate([dl.j1a, dl.j2b, dl.j3a, dl.j3b]).astype(np.int32)
            self.maps.append(torch.from_numpy(m).to(device))
            vs, ve = geom.corner_mode_vectors(dl.axis)
            self.vmode.append(torch.from_numpy(np.concatenate([vs, ve])).to(device))
            self.Ie.append(torch.from_numpy(np.ascontiguousarray(dl.I_e, dtype=np.int32)).to(device))
        self.root_Ie = torch.from_numpy(np.ascontiguousarray(lay.root_I_e, dtype=np.int64)).to(device)
        blob, idx, pmax = geom.device_constants()
        self.leaf_consts = torch.from_numpy(blob).to(device)
        self.leaf_idx = torch.from_numpy(idx).to(device)
        self.probe_max = pmax


@dataclass
class BuildInputs:
    """Host-prepared, device-resident inputs of one build (coefficient samples of the group
    representatives, leaf->group map, layout tables). `build_device` consumes it with no host
    work besides kernel enqueues."""

    tree: object
    nodeset: object
    coeffs: object
    layout: object
    geom: LeafGeometry
    dev_layout: object
    reps: np.ndarray
    gid: np.ndarray
    gid_dev: object
    fields_dev: list
    scalars: tuple
    device: object
    uploaded_bytes: int = 0  # H2D bytes prepare() moved (full sample arrays, before grouping)

    @property
    def ngroups(self):
        return int(self.reps.size)

    def h2d_bytes(self):
        if self.uploaded_bytes:
            return int(self.uploaded_bytes)
        return int(sum(t.numel() * t.element_size() for t in self.fields_dev if t is not None)
                   + self.gid_dev.numel() * 4)

    def device_tensors(self):
        return [t for t in self.fields_dev if t is not None] + [self.gid_dev]


def prepare(tree, nodeset, coeffs, *, device=None, pinned=False):
    """Sample the coefficients on every leaf grid, group bitwise-equal leaves and upload the group
    representatives' samples (solver.py:184-222). Host work + H2D only."""
    torch = _torch()
    lay = layout_of(tree)
    q = lay.q
    if q < 3:
        raise ValueError("p must be >= 3 (need an interior node)")
    geom = LeafGeometry.get(q, tree.leaf_width, tree.leaf_height)
    n_leaf = 1 << (2 * lay.L)
    host_bufs = []
    pinned = pinned and torch.cuda.is_available()

    def pinned_out(shape):  # sample straight into page-locked memory (no staging copy)
        t = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        host_bufs.append(t)
        return t.numpy()

    fields = _sample(coeffs, lay, geom, out=pinned_out if pinned else None)  # ValueError on non-finite samples
    _native.require_device()
    device = torch.device(device if device is not None else "cuda")
    dl = _DeviceLayout.get(lay, geom, device)
    names = [n for n in COEFF_NAMES if not np.isscalar(fields[n])]
    full = {}
    for name in names:
        v = fields[name]
        h = next((t for t in host_bufs if t.numpy().ctypes.data == v.ctypes.data), None) if pinned else None
        if h is None:
            h = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64) if v.flags.writeable
                                 else np.array(v, dtype=np.float64, order="C"))
        full[name] = h.to(device, non_blocking=pinned)
    # group bitwise-equal leaves on the device (host fallback on a hash collision)
    grouped = _group_device([full[n] for n in names], n_leaf) if names else None
    if grouped is not None:
        reps_dev, gid_dev64 = grouped
        reps, gid = reps_dev.cpu().numpy(), gid_dev64.cpu().numpy()
        gid_dev = gid_dev64.to(torch.int32)
    else:
        reps, gid = _group(fields, n_leaf)
        reps_dev = torch.from_numpy(reps).to(device)
        gid_dev = torch.from_numpy(gid.astype(np.int32)).to(device)
    fields_dev, scalars = [], []
    for name in COEFF_NAMES:
        if name not in full:
            fields_dev.append(None)
            scalars.append(float(fields[name]))
        else:
            t = full[name]
            fields_dev.append(t if reps.size == n_leaf else t.index_select(0, reps_dev))
            scalars.append(0.0)
    up = sum(t.numel() * 8 for t in full.values())
    return BuildInputs(tree, nodeset, coeffs, lay, geom, dl, reps, gid, gid_dev, fields_dev, tuple(scalars), device,
                       uploaded_bytes=int(up))


def _ahead_params():
    """(min parent n3, work bound) of the look-ahead interface inverse (hps_merge_level_ahead).

    It pays where the parent's inverse is a latency chain that leaves the GPU idle: about
    0.11 ms per 128 rows (n3 / 128 sequential Gauss-Jordan panels plus small GEMMs, measured).
    Forming X early costs 4 pn3^2 n3 P extra flops (P parents, n3 = this depth's interface), about
    pn3 n3 P * 4 pn3 / 30 TF/s. Look ahead when that is under half the chain it hides:
    pn3 * n3 * P <= 3.2e6. In practice: every depth of L <= 7 trees, none at L >= 8 (measured
    cfg2 14.1 -> 13.45 ms, cfg3 41.9 -> 39.6 ms, cfg4 363.9 -> 366.2 ms had it been on)."""
    import os
    lo = os.environ.get("HPS_AHEAD_MIN_N3")
    work = os.environ.get("HPS_AHEAD_WORK")
    return (int(lo) if lo else 128), (float(work) if work else 3.2e6)


def lookahead_depths(lay):
    """Depths d whose merge stage also forms and inverts the parent depth's (d - 1) interface
    matrix (hps_merge_level_ahead), by the rule of _ahead_params."""
    ahead_min, ahead_work = _ahead_params()
    out = set()
    if ahead_min <= 0:
        return out
    for d in range(1, len(lay.depths)):
        pl, dl_ = lay.depths[d - 1], lay.depths[d]
        if pl.n3 >= ahead_min and float(pl.n3) * dl_.n3 * pl.n_boxes <= ahead_work:
            out.add(d)
    return out


def build_device(inp, *, keep_level_T=False, timeline=None, eps=1e-10, switch_threshold=math.inf,
                 hbs_leaf_size=64, stage_begin=None, ctx=None, pivoted=()):
    """Enqueue the leaf stage and every merge level on the current stream (no host sync).
    `stage_begin(name)`, if given, is called before each stage ("leaf", "merge_d<d>"): BuildGraph
    uses it to capture one CUDA graph per stage. `ctx` is the library context (_native.Context;
    default: slot 0 of the current device); builds in flight at the same time need different ones.
    `pivoted`: depths whose interface systems (n3 > 128) are factored by the pivoted LU instead of
    the residual-checked block inverse (check_build returns the depths whose check failed)."""
    if stage_begin is not None:
        stage_begin("leaf")
    torch = _torch()
    lib = _native.load()
    lay, geom, dl, device = inp.layout, inp.geom, inp.dev_layout, inp.device
    q, L = lay.q, lay.L
    p = q
    n_leaf = 1 << (2 * L)
    p2, ni, nb, ng = p * p, (p - 2) ** 2, 4 * (p - 1), 4 * p
    ngroups = inp.ngroups
    stream = _native.stream_ptr()
    cx = ctx if ctx is not None else _native.context()

    # ---- leaf stage (solver.py:184-247) ----
    fptr = (ctypes_vp * 6)()
    scal = (ctypes_d * 6)()
    for f in range(6):
        t = inp.fields_dev[f]
        fptr[f] = None if t is None else _native.ptr(t).value
        scal[f] = inp.scalars[f]
    Psi = torch.empty((ngroups, ni, nb), dtype=torch.float64, device=device)
    Tleaf = torch.empty((ngroups, ng, ng), dtype=torch.float64, device=device)
    cond = torch.empty(ngroups, dtype=torch.float64, device=device)
    wsb = lib.hps_leaf_workspace_bytes(cx, p, ngroups)
    ws = torch.empty(wsb, dtype=torch.uint8, device=device)
    mark = _marker(timeline, "leaf")
    _native.check(lib.hps_leaf_stage(cx, p, ngroups, fptr, scal, _native.ptr(dl.leaf_consts), _native.ptr(dl.leaf_idx),
                                     dl.probe_max, _native.ptr(Psi), _native.ptr(Tleaf), _native.ptr(cond),
                                     _native.ptr(ws), wsb, stream), "hps_leaf_stage")
    mark()
    del ws
    chunk = max(1, int(2e8 / (8 * p2 * p2)))  # reference chunking, for counter parity (solver.py:226)
    instrumentation.bump("leaf_dtn", -(-ngroups // chunk))

    # ---- merges, deepest depth first (solver.py:266-285) ----
    status = torch.full((max(2 * L, 1),), -1, dtype=torch.int32, device=device)
    S_levels = [None] * (2 * L)
    level_T = [None] * (2 * L) if keep_level_T else None
    child_T, child_stride, child_idx = Tleaf, ng * ng, inp.gid_dev
    # Look-ahead interface inverse (hps_merge_level_ahead): depth d forms, deflates and inverts the
    # parent depth's X beside its own T GEMM (rule in _ahead_params; HPS_AHEAD_MIN_N3=0 disables).
    # The parent's workspace is allocated one depth early.
    ahead = lookahead_depths(lay)
    pivoted = frozenset(pivoted)
    ws_next, pre_inv = None, False
    for d in range(2 * L - 1, -1, -1):
        if stage_begin is not None:
            stage_begin(f"merge_d{d}")
        dlay = lay.depths[d]
        nbatch, n3, ne, m = dlay.n_boxes, dlay.n3, dlay.ne, dlay.m
        S = torch.empty((nbatch, n3, ne), dtype=torch.float64, device=device)
        T = torch.empty((nbatch, ne, ne), dtype=torch.float64, device=device)
        wsb = lib.hps_merge_workspace_bytes(nbatch, n3, ne)
        ws = ws_next if ws_next is not None else torch.empty(wsb, dtype=torch.uint8, device=device)
        ws_next = None
        status_d = ctypes_vp(status.data_ptr() + 4 * d)
        mark = _marker(timeline, f"merge_d{d}")
        pl = lay.depths[d - 1] if d > 0 else None
        if pl is not None and d in ahead:
            pwsb = lib.hps_merge_workspace_bytes(pl.n_boxes, pl.n3, pl.ne)
            ws_next = torch.empty(pwsb, dtype=torch.uint8, device=device)
            _native.check(lib.hps_merge_level_ahead(
                cx, nbatch, n3, ne, m, q, _native.ptr(child_T), child_stride, _native.ptr(child_idx),
                _native.ptr(dl.maps[d]), _native.ptr(dl.vmode[d]), _native.ptr(S), _native.ptr(T), _native.ptr(ws),
                wsb, status_d, 0, int(pre_inv), _native.ptr(dl.maps[d - 1]), pl.n3, pl.ne,
                _native.ptr(dl.vmode[d - 1]), _native.ptr(ws_next), pwsb, ctypes_vp(status.data_ptr() + 4 * (d - 1)),
                0, _merge_flags(d, pivoted), stream), f"hps_merge_level_ahead(depth {d})")
            next_pre = True
        else:
            _native.check(lib.hps_merge_level_ahead(
                cx, nbatch, n3, ne, m, q, _native.ptr(child_T), child_stride, _native.ptr(child_idx),
                _native.ptr(dl.maps[d]), _native.ptr(dl.vmode[d]), _native.ptr(S), _native.ptr(T), _native.ptr(ws),
                wsb, status_d, 0, int(pre_inv), None, 0, 0, None, None, 0, None, 0, _merge_flags(d, pivoted), stream),
                f"hps_merge_level(depth {d})")
            next_pre = False
        pre_inv = next_pre
        mark()
        del ws
        instrumentation.bump("merge", nbatch)
        S_levels[d] = S
        if keep_level_T:
            level_T[d] = T
        child_T, child_stride, child_idx = T, ne * ne, None
    root_dev = child_T[0] if L > 0 else Tleaf[int(inp.gid[0])]

    state = SolverState(
        tree=inp.tree, nodes=inp.nodeset, coeffs=inp.coeffs, q=q, eps=eps, switch_threshold=switch_threshold,
        hbs_leaf_size=hbs_leaf_size, geometry=geom, psi=_LazyPsi(Psi, inp.gid, n_leaf - 1),
        S=_LazyS(S_levels, L), root_T=DtnOperator(device_tensor=root_dev),
        rank_stats={"max_rank": 0, "min_rank": None, "per_level": {}, "n_hbs_matrices": 0},
        n_leaf_groups=ngroups, layout=lay, S_levels=S_levels, Ie_levels=dl.Ie, psi_groups=Psi,
        T_leaf_groups=Tleaf, leaf_group=inp.gid, root_Ie_dev=dl.root_Ie, device=device, level_T=level_T)
    state._status = status
    state._cond = cond
    state._reps = inp.reps
    state._pivoted = pivoted
    return state


def _merge_flags(d, pivoted):
    return (_native.HPS_MERGE_PIVOTED if d in pivoted else 0) | \
        (_native.HPS_MERGE_PARENT_PIVOTED if d - 1 in pivoted else 0)


def build(tree, nodeset, coeffs, eps=1e-10, switch_threshold=2000, hbs_leaf_size=64, *, device=None,
          keep_level_T=False, check=True, timeline=None):
    """One bottom-up sweep producing every operator needed for solves (solver.py:250-289).

    Dense on the GPU regardless of `switch_threshold` (the reference's HBS branch is out of
    scope). With check=False the device status words are not read back (no host sync); call
    `check_build(state)` later to raise the reference's exceptions. `timeline` (a list) receives
    (stage, start_event, end_event) CUDA event pairs for a per-stage breakdown.
    """
    if switch_threshold is None:
        switch_threshold = math.inf
    inp = prepare(tree, nodeset, coeffs, device=device)
    kw = dict(keep_level_T=keep_level_T, timeline=timeline, eps=eps, switch_threshold=switch_threshold,
              hbs_leaf_size=hbs_leaf_size)
    state = build_device(inp, **kw)
    if check:
        state = checked(state, inp, **kw)
    return state


def checked(state, inp, **build_kw):
    """check_build, and where a depth's residual check failed, rebuild with those depths on the
    pivoted LU (at most once per depth) until every check passes. Returns the final state."""
    pivoted = set(getattr(state, "_pivoted", ()))
    while True:
        retry = check_build(state) - pivoted
        if not retry:
            return state
        pivoted |= retry
        instrumentation.bump("pivoted_rebuild")
        state = build_device(inp, pivoted=pivoted, **build_kw)


def _marker(timeline, name):
    """Record a CUDA event now; the returned callable records the end event."""
    if timeline is None:
        return lambda: None
    torch = _torch()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()

    def end():
        e1.record()
        timeline.append((name, e0, e1))
    return end


def check_build(state):
    """Read back the device status words and raise the reference's exceptions (one host sync).
    Returns the set of depths whose fast interface inverse failed its residual check (to rebuild
    with pivoted=...; `build` and `checked` do that); empty normally."""
    return _raise_from_status(state, state._cond.cpu().numpy(), state._status.cpu().numpy())


def _raise_from_status(state, cond, st):
    bad = np.flatnonzero(cond > RESONANCE_COND)
    if bad.size:  # first group in first-occurrence order (solver.py:235-239)
        j = int(bad[0])
        leaf_index = (1 << (2 * state.layout.L)) - 1 + int(state._reps[j])
        raise LeafResonanceError(box=leaf_index, cond=float(cond[j]))
    retry = {d for d in range(len(st)) if st[d] >= _native.HPS_STATUS_PIVOT}
    for d in range(len(st) - 1, -1, -1):  # reference merges deepest (highest index) first
        if 0 <= st[d] < _native.HPS_STATUS_PIVOT and not retry:
            raise MergeResonanceError(box=(1 << d) - 1 + int(st[d]), detail="non-finite solution operator")
    return retry


# ----------------------------------------------------------------------------------------------
# Solve (solver.py:292-316)
# ----------------------------------------------------------------------------------------------
def _boundary_values(state, f):
    ids = state.layout.root_I_e
    if callable(f):
        pts = state.nodes.points[ids]
        return np.asarray(f(pts[:, 0], pts[:, 1]), dtype=float)
    vals = np.asarray(f, dtype=float)
    if vals.shape[:1] != (ids.size,) or vals.ndim > 2:
        raise ValueError(f"boundary data must have length {ids.size}")
    return vals


def rhs_ld(b):
    """Leading dimension of the node-major solution buffer for b right-hand sides."""
    return 1 if b == 1 else -(-b // 8) * 8


def solve_device(state, F, out=None, ctx=None):
    """Device-resident batched solve. F: torch (|Gamma|, b) or (|Gamma|,) fp64 on the device, in
    root.I_e order. Returns U (N, ldu) on the device; columns [:b] are the solutions."""
    torch = _torch()
    lib = _native.load()
    cx = ctx if ctx is not None else _native.context()
    lay = state.layout
    if F.dim() == 1:
        F = F[:, None]
    b = F.shape[1]
    ldu = rhs_ld(b)
    N = lay.N
    # Every row of U is written: the boundary rows [0, n_gamma) by the scatter of F (root.I_e is a
    # permutation of them) and every interface range by its depth's solve (TreeLayout.depth_off), so
    # only the padding columns of a batch that is not a multiple of 8 need zeros (the GEMM path
    # reads them as right-hand sides).
    if out is None:
        U = (torch.empty if ldu == b else torch.zeros)((N, ldu), dtype=torch.float64, device=state.device)
    else:
        U = out
        if ldu != b:
            U.zero_()
    U[:, :b].index_copy_(0, state.root_Ie_dev, F.to(torch.float64))
    stream = _native.stream_ptr()
    for d in range(2 * lay.L):
        dl = lay.depths[d]
        nrhs = b if b <= 8 else ldu
        _native.check(lib.hps_solve_level(cx, dl.n_boxes, dl.n3, dl.ne, _native.ptr(state.S_levels[d]),
                                          _native.ptr(state.Ie_levels[d]), int(lay.depth_off[d]),
                                          _native.ptr(U), ldu, nrhs, stream), f"hps_solve_level(depth {d})")
    return U


def solve(state, f):
    """Solution at every tabulation node (solver.py:303-316). `f` is a callable, a vector in
    root.I_e order, or an (|Gamma|, b) batch (returns (N, b))."""
    torch = _torch()
    instrumentation.bump("solve")
    vals = _boundary_values(state, f)
    single = vals.ndim == 1
    F = torch.from_numpy(np.ascontiguousarray(vals if not single else vals[:, None])).to(state.device)
    U = solve_device(state, F)
    u = U[:, :F.shape[1]].cpu().numpy()
    return u[:, 0].copy() if single else u


class Pipeline:
    """Build + solve a stream of problems on one discretisation with host and device overlapped.

    The reference builds and solves one problem per `build`/`solve` call (solver.py:170-316); a
    service answering many coefficient fields / boundary data on the same tree runs that pair in a
    loop. Here, while the device builds and solves problem i on the main stream, a host thread
    samples, uploads and groups problem i+1's coefficients (`prepare`, pinned memory, its own
    stream), and problem i-1's u and status words come back on a third stream. With streams=2
    (default up to L = 8) problems alternate between two compute streams, so problem i's
    latency-bound top merges run beside problem i+1's leaf stage. Every problem still makes its
    own H2D copies and its own D2H of u; at most three states are alive at once.

    `run(jobs)` takes an iterable of (coeffs, F), F a host (|Gamma|, b) or (|Gamma|,) array in
    root.I_e order, and yields (U, state) per job in order: U is a pinned host tensor (N, ldu) whose
    columns [:b] are the solutions, state the SolverState (valid until the caller drops it)."""

    def __init__(self, tree, nodeset, *, device=None, overlap_results=True, reuse_graphs=False, streams=None):
        torch = _torch()
        _native.require_device()
        self.overlap_results = overlap_results
        # reuse_graphs: build + solve replayed from two alternating BuildGraph captures (keyed by the
        # group count, coefficient structure and batch width; other jobs run eagerly). A yielded
        # state then lives in graph memory and is valid until the next item is requested.
        self.reuse_graphs = reuse_graphs
        self._graphs = [{} for _ in range(4)]
        self._jobs = 0
        self.tree, self.nodeset = tree, nodeset
        self.device = torch.device(device if device is not None else "cuda")
        # the next problem's uploads and grouping kernels run beside the current build: highest
        # stream priority, so they take SM slots as soon as any free up
        import os as _os
        prio = int(_os.environ.get("HPS_UPLOAD_PRIORITY", "1"))
        self._upload = torch.cuda.Stream(self.device, priority=-prio if prio else 0)
        # streams=2: consecutive problems are built and solved on two alternating compute streams,
        # so one problem's latency-bound top merges (interface inverses on a few CTAs) overlap the
        # next problem's leaf stage. Each problem waits for the D2H of the problem two before it
        # (the previous user of its graph slot / workspace).
        # Default: two streams up to L = 8 (cfg2 e2e 15.0 -> 13.2 ms/problem, cfg3 41.5 -> 37.6 ms);
        # one at L >= 9, where two problems' operators in flight would not fit beside each other.
        if streams is None:
            env = _os.environ.get("HPS_PIPE_STREAMS")
            streams = int(env) if env else (2 if getattr(getattr(tree, "layout", tree), "L", 0) <= 8 else 1)
        self._mains = [torch.cuda.Stream(self.device) for _ in range(max(1, min(4, int(streams))))]
        self._nslots = max(2, len(self._mains))  # graph / scratch / workspace slots, used round robin
        self._main = self._mains[0]
        self._slot_done = [None] * 4
        self._d2h = torch.cuda.Stream(self.device)
        import concurrent.futures
        self._host = concurrent.futures.ThreadPoolExecutor(max_workers=1)

    def _prepare(self, coeffs):
        torch = _torch()
        with torch.cuda.device(self.device), torch.cuda.stream(self._upload):
            inp = prepare(self.tree, self.nodeset, coeffs, device=self.device, pinned=True)
            ready = torch.cuda.Event()
            ready.record(self._upload)
        return inp, ready

    def run(self, jobs):
        torch = _torch()
        it = iter(jobs)
        job = next(it, None)
        fut = self._host.submit(self._prepare, job[0]) if job is not None else None
        pending = None
        while fut is not None:
            k = self._jobs  # job counter across run() calls: stream, graph slot and scratch slot
            inp, ready = fut.result()
            nxt = next(it, None)
            F = job[1]
            fut = self._host.submit(self._prepare, nxt[0]) if nxt is not None else None
            main = self._mains[k % len(self._mains)]
            with torch.cuda.device(self.device):
                with torch.cuda.stream(main):
                    main.wait_event(ready)
                    sl = k % self._nslots
                    if len(self._mains) > 1 and self._slot_done[sl] is not None:
                        main.wait_event(self._slot_done[sl])
                    for t in inp.device_tensors():
                        t.record_stream(main)
                    Fh = F if torch.is_tensor(F) else torch.from_numpy(np.ascontiguousarray(np.asarray(F, dtype=float)))
                    if Fh.dim() == 1:
                        Fh = Fh[:, None]
                    if not Fh.is_pinned():
                        Fh = Fh.pin_memory()
                    Fd = Fh.to(self.device, non_blocking=True)
                    # this job's library context (its own side streams and split-K scratch: the
                    # neighbouring job on the other stream may still be running)
                    cx = _native.context(sl if len(self._mains) > 1 else 0, self.device)
                    g = self._graph_for(inp, Fd.shape[1], sl) if self.reuse_graphs else None
                    if g is not None:
                        g.load(inp, Fd)
                        st = g.replay_build()
                        U = g.replay_solve()
                    else:
                        st = build_device(inp, ctx=cx)
                        U = solve_device(st, Fd, ctx=cx)
                    st._job = (inp, Fd)  # for a pivoted rebuild (_finish)
                    solved = torch.cuda.Event()
                    solved.record(main)
                # results and status words come back on their own stream, so the next job's build
                # is enqueued on the main stream before this job's D2H is waited for
                with torch.cuda.stream(self._d2h):
                    self._d2h.wait_event(solved)
                    outs = []
                    for t in (U, st._cond, st._status):
                        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                        h.copy_(t, non_blocking=True)
                        t.record_stream(self._d2h)
                        outs.append(h)
                    done = torch.cuda.Event()
                    done.record(self._d2h)
                    self._slot_done[sl] = done
            self._jobs += 1
            del U
            if pending is not None:
                yield self._finish(*pending)
            pending = (st, outs, done)
            del st
            if not self.overlap_results:
                yield self._finish(*pending)
                pending = None
            job = nxt
        if pending is not None:
            yield self._finish(*pending)

    def _graph_for(self, inp, nrhs, sidx):
        slot = self._graphs[sidx]
        key = (inp.ngroups, tuple(t is not None for t in inp.fields_dev), tuple(inp.scalars), int(nrhs))
        g = slot.get(key)
        if g is None:
            if len(slot) >= 4:  # bound the captured memory
                slot.clear()
            torch = _torch()
            try:
                g = slot[key] = BuildGraph(inp, nrhs=nrhs, ctx_slot=sidx if len(self._mains) > 1 else 0)
            except torch.OutOfMemoryError:  # two captured states do not fit: stay eager from here on
                slot.clear()
                self._graphs = [{} for _ in range(4)]
                self.reuse_graphs = False
                torch.cuda.empty_cache()
                return None
        return g

    def _finish(self, st, outs, done):
        done.synchronize()
        U_host, cond, status = outs
        retry = _raise_from_status(st, cond.numpy(), status.numpy())
        if retry:
            # a fast interface inverse failed its residual check: rebuild this job with the pivoted
            # LU at those depths and solve again (eager, on the main stream; rare)
            torch = _torch()
            inp, Fd = st._job
            with torch.cuda.device(self.device), torch.cuda.stream(self._main):
                st = checked(build_device(inp, pivoted=retry), inp)
                U_host = solve_device(st, Fd).cpu()
        instrumentation.bump("solve")
        return U_host, st

    def close(self):
        self._host.shutdown(wait=True)


class BuildGraph:
    """One build (and optionally one batched solve) captured into CUDA graphs and replayed.

    For loops that rebuild the same discretisation with new coefficient samples (time stepping,
    parameter sweeps, benchmarks): the ~290 kernel launches of a build become one graph launch per
    stage (the leaf stage and each merge depth) plus one for the solve. That removes the launch
    gaps, which dominate the small, latency-bound top merges, and keeps per-stage event timing
    possible between the replays.

    `BuildGraph(inp, nrhs)` captures for inputs shaped like `inp` (same tree, same number of leaf
    groups, same non-constant coefficient fields and constant values). `run(inp, F)` copies the
    new inputs into the graphs' static buffers, replays, and returns (state, U): both live in
    the graphs' memory pool and are overwritten by the next run. `check_build(state)` works as
    usual. Replays enqueue on the current stream. `launches` is the number of library kernel
    launches one build + solve replay performs."""

    _warmed = set()

    def __init__(self, inp, nrhs=0, ctx_slot=0, pivoted=()):
        torch = _torch()
        lib = _native.load()
        # the library context (side streams, split-K scratch) this capture bakes in: two graphs
        # replayed at once on two streams need different ones, see Pipeline(streams=2)
        self.ctx_slot = int(ctx_slot)
        self.ctx = _native.context(self.ctx_slot, inp.device)
        # depths on the pivoted LU (check_build's answer when a residual check failed)
        self.pivoted = frozenset(pivoted)
        self.torch = torch
        self.layout, self.ngroups, self.scalars = inp.layout, inp.ngroups, tuple(inp.scalars)
        self._present = tuple(t is not None for t in inp.fields_dev)
        fields = [None if t is None else t.clone() for t in inp.fields_dev]
        self._inp = BuildInputs(inp.tree, inp.nodeset, inp.coeffs, inp.layout, inp.geom, inp.dev_layout,
                                inp.reps, inp.gid, inp.gid_dev.clone(), fields, tuple(inp.scalars), inp.device)
        self.nrhs = int(nrhs)
        self._F = (torch.zeros((len(inp.layout.root_I_e), self.nrhs), dtype=torch.float64, device=inp.device)
                   if self.nrhs else None)
        side = torch.cuda.Stream(inp.device)
        side.wait_stream(torch.cuda.current_stream())
        pool = torch.cuda.graph_pool_handle()
        self.stages = []
        n0 = lib.hps_launch_count()
        key = (id(inp.layout), inp.ngroups, self._present, self.scalars, self.nrhs, self.ctx_slot, self.pivoted)
        with torch.cuda.stream(side):
            if key not in BuildGraph._warmed:
                # warm-up: lazy attributes and scratch sizes outside the capture (once per shape)
                st = build_device(self._inp, ctx=self.ctx, pivoted=self.pivoted)
                if self.nrhs:
                    solve_device(st, self._F, ctx=self.ctx)
                del st
                torch.cuda.synchronize()
                torch.cuda.empty_cache()  # the warm-up state's memory (L=9: ~50 GB) back before the capture
                BuildGraph._warmed.add(key)
            n0 = lib.hps_launch_count()

            # thread_local: other host threads (the Pipeline's preparation thread) may sync or
            # allocate pinned memory meanwhile without invalidating this capture
            self.stage_launches = []

            def begin(name):
                if self.stages:
                    self.stages[-1][1].capture_end()
                    self.stage_launches.append(int(lib.hps_launch_count() - self._l0))
                g = torch.cuda.CUDAGraph()
                self._l0 = lib.hps_launch_count()
                g.capture_begin(pool=pool, capture_error_mode="thread_local")
                self.stages.append((name, g))

            active = [None]

            def begin_tracked(name):
                begin(name)
                active[0] = self.stages[-1][1]

            try:
                self.state = build_device(self._inp, stage_begin=begin_tracked, ctx=self.ctx, pivoted=self.pivoted)
                self.stages[-1][1].capture_end()
                self.stage_launches.append(int(lib.hps_launch_count() - self._l0))
                active[0] = None
                self.solve_graph, self.U = None, None
                if self.nrhs:
                    self.solve_graph = torch.cuda.CUDAGraph()
                    self.solve_graph.capture_begin(pool=pool, capture_error_mode="thread_local")
                    active[0] = self.solve_graph
                    self.U = solve_device(self.state, self._F, ctx=self.ctx)
                    self.solve_graph.capture_end()
                    active[0] = None
            except BaseException:
                if active[0] is not None:  # leave the stream out of capture mode before re-raising
                    try:
                        active[0].capture_end()
                    except BaseException:
                        pass
                self.stages, self.state = [], None
                raise
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.launches = int(lib.hps_launch_count() - n0)

    def matches(self, inp):
        return (inp.layout is self.layout and inp.ngroups == self.ngroups and tuple(inp.scalars) == self.scalars
                and tuple(t is not None for t in inp.fields_dev) == self._present)

    def load(self, inp=None, F=None):
        """Copy new inputs (and boundary data) into the static buffers (stream-ordered)."""
        if inp is not None:
            if not self.matches(inp):
                raise ValueError("BuildGraph: inputs differ in layout, group count or coefficient structure")
            for dst, src in zip(self._inp.fields_dev, inp.fields_dev):
                if dst is not None:
                    dst.copy_(src, non_blocking=True)
            self._inp.gid_dev.copy_(inp.gid_dev, non_blocking=True)
            st = self.state
            st._reps, st.leaf_group, st.coeffs = inp.reps, inp.gid, inp.coeffs
            st.psi = _LazyPsi(st.psi_groups, inp.gid, (1 << (2 * self.layout.L)) - 1)
            st._gid_dev = None
        if F is not None:
            if not self.nrhs:
                raise ValueError("BuildGraph: captured without a solve (nrhs=0)")
            Ft = F if self.torch.is_tensor(F) else self.torch.from_numpy(np.ascontiguousarray(F, dtype=np.float64))
            self._F.copy_(Ft.reshape(self._F.shape), non_blocking=True)

    def replay_build(self, timeline=None):
        """Replay the build stages; with `timeline` (a list), append (name, start, end) events."""
        for name, g in self.stages:
            if timeline is None:
                g.replay()
            else:
                e0 = self.torch.cuda.Event(enable_timing=True)
                e1 = self.torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                timeline.append((name, e0, e1))
        return self.state

    def replay_solve(self):
        if self.solve_graph is None:
            raise ValueError("BuildGraph: captured without a solve (nrhs=0)")
        self.solve_graph.replay()
        return self.U

    def run(self, inp=None, F=None):
        self.load(inp, F)
        self.replay_build()
        U = self.replay_solve() if self.solve_graph is not None else None
        return self.state, U


def apply_global_dtn(state, f):
    """Root DtN applied to boundary data (solver.py:319-327), on the device."""
    torch = _torch()
    lib = _native.load()
    instrumentation.bump("apply_dtn")
    vals = _boundary_values(state, f)
    single = vals.ndim == 1
    V = vals[:, None] if single else vals
    n, b = V.shape
    ld = -(-b // 2) * 2
    F = torch.zeros((n, ld), dtype=torch.float64, device=state.device)
    F[:, :b] = torch.from_numpy(np.ascontiguousarray(V)).to(state.device)
    out = torch.empty((n, ld), dtype=torch.float64, device=state.device)
    Tr = state.root_T.device_tensor
    _native.check(lib.hps_dgemm_batched(_native.context(), n, ld, n, 1, 1.0, _native.ptr(Tr), n, 0, _native.ptr(F), ld,
                                        0, None, 0, 0.0, _native.ptr(out), ld, 0, _native.stream_ptr()),
                  "hps_dgemm_batched")
    r = out[:, :b].cpu().numpy()
    return r[:, 0].copy() if single else r


# ----------------------------------------------------------------------------------------------
# Post-processing on the device (solver.py:330-400): per-leaf Chebyshev
# fields from the solution (hps_leaf_fields), point evaluation (hps_eval_points), and the
# gauge-fixed Gauss-node solution re-tabulated from the fields (hps_gauge_sides / _gather).
# ----------------------------------------------------------------------------------------------
class _PostTables:
    """Per-(layout, geometry, device) tables of the post-processing kernels."""

    _cache = {}

    @classmethod
    def get(cls, lay, geom, device):
        key = (id(lay), geom.p, geom.width, geom.height, str(device))
        v = cls._cache.get(key)
        if v is None:
            v = cls._cache[key] = cls(lay, geom, device)
        return v

    def __init__(self, lay, geom, device):
        torch = _torch()
        dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)
        self.leaf_Ie = dev(lay.leaf_I_e, np.int32)
        self.L1 = dev(geom.L1, np.float64)
        self.J_i = dev(geom.J_i, np.int32)
        self.J_e = dev(geom.J_e, np.int32)
        self.Qx = dev(geom.Qx, np.float64)
        self.Qy = dev(geom.Qy, np.float64)
        # owners of every node: rows leaf * 4q + k of the side table; outer-boundary nodes have one
        # owner and keep the Dirichlet data (src -1)
        flat = np.ascontiguousarray(lay.leaf_I_e).reshape(-1)
        order = np.argsort(flat, kind="stable")
        counts = np.bincount(flat, minlength=lay.N)
        start = np.concatenate([[0], np.cumsum(counts)[:-1]])
        src = np.full((lay.N, 2), -1, dtype=np.int32)
        two = counts == 2
        src[two, 0] = order[start[two]]
        src[two, 1] = order[start[two] + 1]
        self.src = dev(src, np.int32)
        cells = np.asarray(lay.leaf_cells)
        n = 1 << lay.L
        self.cell_leaf = np.empty((n, n), dtype=np.int64)
        self.cell_leaf[cells[:, 0], cells[:, 1]] = np.arange(cells.shape[0])


def _gid_dev(state):
    g = getattr(state, "_gid_dev", None)
    if g is None:
        torch = _torch()
        g = torch.from_numpy(np.ascontiguousarray(state.leaf_group, dtype=np.int32)).to(state.device)
        state._gid_dev = g
    return g


def _solution_device(state, u):
    """(U device (N, ld), nrhs, single) from a host vector/batch or a device solve output."""
    torch = _torch()
    if torch.is_tensor(u):
        U = u if u.dim() == 2 else u[:, None]
        if U.device.type != "cuda":
            U = U.to(state.device)
        return U.contiguous().to(torch.float64), U.shape[1], u.dim() == 1
    a = np.asarray(u, dtype=float)
    single = a.ndim == 1
    a = a[:, None] if single else a
    if a.shape[0] != state.layout.N:
        raise ValueError(f"solution must have {state.layout.N} rows")
    return torch.from_numpy(np.ascontiguousarray(a)).to(state.device), a.shape[1], single


def _leaf_fields_dev(state, U, nrhs, leaves):
    torch = _torch()
    lib = _native.load()
    tb = _PostTables.get(state.layout, state.geometry, state.device)
    p = state.geometry.p
    lv = torch.from_numpy(np.ascontiguousarray(leaves, dtype=np.int32)).to(state.device)
    W = torch.empty((len(leaves), p * p, nrhs), dtype=torch.float64, device=state.device)
    _native.check(lib.hps_leaf_fields(len(leaves), p, _native.ptr(U), U.shape[1], nrhs, _native.ptr(lv),
                                      _native.ptr(tb.leaf_Ie), _native.ptr(_gid_dev(state)), _native.ptr(tb.L1),
                                      _native.ptr(state.psi_groups), _native.ptr(tb.J_i), _native.ptr(tb.J_e),
                                      _native.ptr(W), _native.stream_ptr()), "hps_leaf_fields")
    return W


def leaf_fields(state, u, leaves=None):
    """p x p Chebyshev field of every (or every listed) leaf, x1-major (solver.py:349-356), on the
    device: (n, p, p) for a vector u, (n, p, p, b) for a batch. Invariant under the interface null
    modes, so it is the gauge-free output of a solve."""
    U, nrhs, single = _solution_device(state, u)
    n_leaf = 1 << (2 * state.layout.L)
    leaves = np.arange(n_leaf) if leaves is None else np.asarray(leaves)
    p = state.geometry.p
    W = _leaf_fields_dev(state, U, nrhs, leaves).view(len(leaves), p, p, nrhs)
    return W[..., 0] if single else W


def _owning_leaves(state, pts):
    """Vectorised _owning_leaf (solver.py:330-346): leaf slot and leaf lower corner per point."""
    tree, lay = state.tree, state.layout
    dom = tree.domain
    x, y = pts[:, 0], pts[:, 1]
    inside = (x >= dom.x_lo) & (x <= dom.x_hi) & (y >= dom.y_lo) & (y <= dom.y_hi)
    if not np.all(inside):
        k = int(np.flatnonzero(~inside)[0])
        raise ValueError(f"target ({x[k]}, {y[k]}) lies outside the domain")
    n = 1 << tree.levels

    def cell(t, extent):
        s_ = (t / extent) * n
        i = np.floor(s_).astype(np.int64)
        i = np.where((i == s_) & (i > 0), i - 1, i)
        return np.clip(i, 0, n - 1)

    ix, iy = cell(x - dom.x_lo, dom.width), cell(y - dom.y_lo, dom.height)
    tb = _PostTables.get(lay, state.geometry, state.device)
    return tb.cell_leaf[ix, iy], lay.xline[ix], lay.yline[iy]


def _eval(state, u, pts, rx, ry, leaf):
    torch = _torch()
    lib = _native.load()
    U, nrhs, single = _solution_device(state, u)
    uniq, slot = np.unique(leaf, return_inverse=True)
    W = _leaf_fields_dev(state, U, nrhs, uniq)
    dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(state.device)
    # the argument tensors must stay referenced until the launch: a temporary freed inside the call
    # expression goes back to the caching allocator and the next one may reuse its block
    slot_d, rx_d, ry_d = dev(slot, np.int32), dev(rx, np.float64), dev(ry, np.float64)
    out = torch.empty((len(pts), nrhs), dtype=torch.float64, device=state.device)
    _native.check(lib.hps_eval_points(len(pts), state.geometry.p, _native.ptr(W), nrhs, _native.ptr(slot_d),
                                      _native.ptr(rx_d), _native.ptr(ry_d), _native.ptr(out), _native.stream_ptr()),
                  "hps_eval_points")
    r = out.cpu().numpy()
    return r[:, 0].copy() if single else r


def post_process(state, u, targets):
    """Solution at arbitrary points via leaf spectral interpolation (solver.py:359-377), on the
    device. u: the solve output (vector, (N, b) batch, or the device tensor of solve_device)."""
    geom = state.geometry
    pts = np.asarray(targets, dtype=float).reshape(-1, 2)
    if pts.shape[0] == 0:
        return np.empty(0)
    leaf, xlo, ylo = _owning_leaves(state, pts)
    rx = interp_matrix(geom.cheb_x, pts[:, 0] - xlo)
    ry = interp_matrix(geom.cheb_y, pts[:, 1] - ylo)
    return _eval(state, u, pts, rx, ry, leaf)


def boundary_flux_at(state, u, targets):
    """Coordinate-derivative flux at outer-boundary points (solver.py:380-400), on the device:
    d/dx1 on the vertical sides, d/dx2 on the horizontal ones (rx Dx W ry^T, rx W (ry Dy)^T)."""
    geom = state.geometry
    dom = state.tree.domain
    pts = np.asarray(targets, dtype=float).reshape(-1, 2)
    if pts.shape[0] == 0:
        return np.empty(0)
    x, y = pts[:, 0], pts[:, 1]
    on_v = (x == dom.x_lo) | (x == dom.x_hi)
    on_h = (y == dom.y_lo) | (y == dom.y_hi)
    if not np.all(on_v | on_h):
        k = int(np.flatnonzero(~(on_v | on_h))[0])
        raise ValueError(f"target ({x[k]}, {y[k]}) is not on the outer boundary")
    leaf, xlo, ylo = _owning_leaves(state, pts)
    rx = interp_matrix(geom.cheb_x, x - xlo)
    ry = interp_matrix(geom.cheb_y, y - ylo)
    dx = on_v & ~on_h
    rx[dx] = rx[dx] @ geom.Dx
    ry[~dx] = ry[~dx] @ geom.Dy
    return _eval(state, u, pts, rx, ry, leaf)


def gauge_fixed_solution(state, u):
    """Gauss-node solution re-tabulated from the leaf Chebyshev fields.

    Every node on a leaf edge takes the mean of its two leaves' side interpolants (the L4 blocks,
    Qx W[:,0], Qy W[p-1,:], Qx W[:,p-1], Qy W[0,:]); outer-boundary nodes keep the Dirichlet data.
    Unlike the raw solve output, whose interface values carry the null-mode gauge,
    this u is a function of the null-mode-invariant fields only. Returns a device tensor (N, b)."""
    torch = _torch()
    lib = _native.load()
    U, nrhs, single = _solution_device(state, u)
    lay, geom = state.layout, state.geometry
    tb = _PostTables.get(lay, geom, state.device)
    n_leaf = 1 << (2 * lay.L)
    W = _leaf_fields_dev(state, U, nrhs, np.arange(n_leaf))
    side = torch.empty((n_leaf, 4 * geom.p, nrhs), dtype=torch.float64, device=state.device)
    _native.check(lib.hps_gauge_sides(n_leaf, geom.p, _native.ptr(W), nrhs, _native.ptr(tb.Qx), _native.ptr(tb.Qy),
                                      _native.ptr(side), _native.stream_ptr()), "hps_gauge_sides")
    out = torch.empty((lay.N, nrhs), dtype=torch.float64, device=state.device)
    _native.check(lib.hps_gauge_gather(lay.N, nrhs, _native.ptr(side), _native.ptr(tb.src), _native.ptr(U), U.shape[1],
                                       _native.ptr(out), nrhs, _native.stream_ptr()), "hps_gauge_gather")
    return out[:, 0] if single else out


def memory_report(state):
    """Deterministic accounting of stored operators, 8 bytes a scalar (solver.py:403-432)."""
    lay = state.layout
    per_level = {d: (1 << d) * lay.depths[d].n3 * lay.depths[d].ne for d in range(2 * lay.L)}
    geom = state.geometry
    ni, nb = (geom.p - 2) ** 2, 4 * (geom.p - 1)
    leaf_entries = state.n_leaf_groups * ni * nb + geom.L1.size + geom.L4.size
    root_entries = state.root_T.n_stored_entries()
    total = root_entries + leaf_entries + sum(per_level.values())
    return {
        "R_mb": total * 8 / 1e6,
        "total_entries": int(total),
        "root_dtn_mb": root_entries * 8 / 1e6,
        "leaf_ops_mb": leaf_entries * 8 / 1e6,
        "solution_ops_mb_per_level": {int(k): v * 8 / 1e6 for k, v in sorted(per_level.items())},
        "rank_stats": {"max_rank": 0, "min_rank": None, "n_hbs_matrices": 0, "per_level": {}},
    }
