"""Multi-GPU build and solve by quadtree subtrees. One process per GPU.

With N = 2^s ranks, rank r owns the box at depth s, slot r (for N = 8: boxes 7..14, a 2 x 4
split of the domain) and everything below it.

* Build: each rank runs the leaf stage for its own leaves and every merge level below depth s,
  with no communication. For the top s depths, the owner of a parent is the owner of its child a
  (the left/bottom one). The owner of child b sends its DtN matrix with one point-to-point
  `send`; the owner merges. The root DtN ends on rank 0. S of a top-depth box stays on its owner.
* Solve: rank 0 holds the boundary batch. Top-down over the top depths, each owner applies its S
  and sends the child-b boundary values u[I_e(child b)] to the owner of child b. Then every rank
  runs its subtree solve independently. The output u stays sharded: rank r owns the
  rows of its subtree (`DistState.owned_rows`). `gather_solution` assembles it on rank 0.

The orchestration is backend-agnostic. `CudaBackend` drives libhps_b200.so on the rank's GPU,
with NCCL as the transport. tests/test_distributed.py runs the same orchestration with a numpy
backend over gloo, world_size 2 and 4, against the single-process oracle.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigError
from .grid import layout_of
from .leafops import LeafGeometry

__all__ = ["CudaBackend", "DistState", "prepare_distributed", "build_distributed", "check_distributed",
           "solve_distributed", "gather_solution", "subtree_plan", "TorchComm", "LocalComm"]


# ----------------------------------------------------------------------------------------------
# Ownership plan (pure integer logic)
# ----------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class SubtreePlan:
    L: int
    world: int
    s: int  # split depth

    def owner(self, d, k):
        """Rank owning box (depth d, slot k)."""
        if d >= self.s:
            return k >> (d - self.s)
        return k << (self.s - d)

    def local_slots(self, rank, d):
        """[lo, hi) slots of depth d (d >= s) inside rank's subtree."""
        w = 1 << (d - self.s)
        return rank * w, (rank + 1) * w

    def top_boxes(self, rank, d):
        """Slots at a top depth d < s that `rank` owns (at most one)."""
        k, rem = divmod(rank, 1 << (self.s - d))
        return [k] if rem == 0 else []


def subtree_plan(L, world):
    s = int(round(math.log2(world))) if world > 0 else -1
    if world < 1 or (1 << s) != world:
        raise ConfigError(f"world size {world} is not a power of two")
    if s > 2 * L:
        raise ConfigError(f"world size {world} exceeds the number of leaves 4^{L}")
    return SubtreePlan(L, world, s)


# ----------------------------------------------------------------------------------------------
# CUDA backend (one GPU per rank)
# ----------------------------------------------------------------------------------------------
class CudaBackend:
    """Stage calls into libhps_b200.so for a subset of slots, on the current CUDA device."""

    def __init__(self, tree, device=None, ctx_slot=0):
        import torch

        from .solver import _DeviceLayout

        _native.require_device()
        self.torch = torch
        self.lib = _native.load()
        self.device = torch.device(device if device is not None else "cuda")
        self.lay = layout_of(tree)
        self.geom = LeafGeometry.get(self.lay.q, tree.leaf_width, tree.leaf_height)
        self.dl = _DeviceLayout.get(self.lay, self.geom, self.device)
        # ranks sharing one device (LocalComm) need their own library context each
        self.ctx = _native.context(ctx_slot, device=self.device)

    # -- tensors / transport --
    def empty(self, shape):
        return self.torch.empty(shape, dtype=self.torch.float64, device=self.device)

    def from_numpy(self, a, dtype=None):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def upload(self, a):
        return a if isinstance(a, self.torch.Tensor) else self.from_numpy(a)

    def to_numpy(self, t):
        return t.cpu().numpy()

    # -- stages --
    def leaf_stage(self, fields_local, scalars, ngroups):
        lib, torch, q = self.lib, self.torch, self.lay.q
        ni, nb, ng = (q - 2) ** 2, 4 * (q - 1), 4 * q
        fptr = (ctypes.c_void_p * 6)()
        scal = (ctypes.c_double * 6)()
        keep = []
        for f in range(6):
            if fields_local[f] is None:
                fptr[f] = None
            else:
                t = self.upload(fields_local[f])
                keep.append(t)
                fptr[f] = _native.ptr(t).value
            scal[f] = scalars[f]
        Psi = self.empty((ngroups, ni, nb))
        T = self.empty((ngroups, ng, ng))
        cond = self.empty((ngroups,))
        wsb = lib.hps_leaf_workspace_bytes(self.ctx, q, ngroups)
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        _native.check(lib.hps_leaf_stage(self.ctx, q, ngroups, fptr, scal, _native.ptr(self.dl.leaf_consts),
                                         _native.ptr(self.dl.leaf_idx), self.dl.probe_max, _native.ptr(Psi),
                                         _native.ptr(T), _native.ptr(cond), _native.ptr(ws), wsb,
                                         _native.stream_ptr()), "hps_leaf_stage")
        return Psi, T, cond

    def merge_level(self, d, nbatch, child_T, child_idx, status, parent_status=None, pivoted=()):
        """One depth's merges for this rank's slots. With `parent_status` (the next call merges
        these boxes' parents on this rank), the look-ahead inverse of solver.build_device runs too
        (hps_merge_level_ahead, where solver.lookahead_depths applies); the next call then starts
        from the pre-inverted interface matrices."""
        from .solver import lookahead_depths

        lib, torch = self.lib, self.torch
        dl = self.lay.depths[d]
        S = self.empty((nbatch, dl.n3, dl.ne))
        T = self.empty((nbatch, dl.ne, dl.ne))
        wsb = lib.hps_merge_workspace_bytes(nbatch, dl.n3, dl.ne)
        pre = getattr(self, "_ahead_ws", None) is not None and self._ahead_ws[0] == (d, nbatch)
        ws = self._ahead_ws[1] if pre else torch.empty(wsb, dtype=torch.uint8, device=self.device)
        self._ahead_ws = None
        idx = None if child_idx is None else self.torch.from_numpy(np.asarray(child_idx, np.int32)).to(self.device)
        if parent_status is not None and nbatch % 2 == 0 and d in lookahead_depths(self.lay):
            pl = self.lay.depths[d - 1]
            pwsb = lib.hps_merge_workspace_bytes(nbatch // 2, pl.n3, pl.ne)
            pws = torch.empty(pwsb, dtype=torch.uint8, device=self.device)
            pargs = (_native.ptr(self.dl.maps[d - 1]), pl.n3, pl.ne, _native.ptr(self.dl.vmode[d - 1]),
                     _native.ptr(pws), pwsb, _native.ptr(parent_status), 0)
            self._ahead_ws = ((d - 1, nbatch // 2), pws)
        else:
            pargs = (None, 0, 0, None, None, 0, None, 0)
        _native.check(lib.hps_merge_level_ahead(self.ctx, nbatch, dl.n3, dl.ne, dl.m, self.lay.q, _native.ptr(child_T),
                                                dl.m * dl.m, _native.ptr(idx), _native.ptr(self.dl.maps[d]),
                                                _native.ptr(self.dl.vmode[d]), _native.ptr(S), _native.ptr(T),
                                                _native.ptr(ws), wsb, _native.ptr(status), 0, int(pre), *pargs,
                                                _merge_flags(d, pivoted), _native.stream_ptr()),
                      f"hps_merge_level(depth {d})")
        return S, T

    # -- split merge of the distributed top depths (hps_merge_interface / _interface_solve / _assemble) --
    def merge_interface(self, d, children, status, pivoted=()):
        """Gathers, deflation and factorisation of one parent's interface system. Returns the
        factored X (inverse for n3 <= 128, L\\U for n3 > 128), its row permutation, R and C."""
        lib, torch = self.lib, self.torch
        dl = self.lay.depths[d]
        n3, ne, m = dl.n3, dl.ne, dl.m
        Xf = self.empty((1, n3, n3))
        perm = torch.empty((1, n3), dtype=torch.int32, device=self.device)
        R = self.empty((1, n3, ne))
        C = self.empty((1, ne, n3))
        wsb = lib.hps_merge_workspace_bytes(1, n3, ne)
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        _native.check(lib.hps_merge_interface(self.ctx, 1, n3, ne, m, self.lay.q, _native.ptr(children), m * m, None,
                                              _native.ptr(self.dl.maps[d]), _native.ptr(self.dl.vmode[d]),
                                              _native.ptr(Xf), _native.ptr(perm), _native.ptr(R), _native.ptr(C),
                                              _native.ptr(ws), wsb, _native.ptr(status), 0,
                                              _merge_flags(d, pivoted), _native.stream_ptr()),
                      f"hps_merge_interface(depth {d})")
        return Xf, perm, R, C

    def interface_solve(self, d, Xf, perm, Rp, status, pivoted=()):
        n3, w = Rp.shape[1], Rp.shape[2]
        Sp = self.empty((1, n3, w))
        _native.check(self.lib.hps_interface_solve(self.ctx, n3, w, 1, _native.ptr(Xf), _native.ptr(perm),
                                                   _native.ptr(Rp), _native.ptr(Sp), _native.ptr(status), 0,
                                                   _merge_flags(d, pivoted), _native.stream_ptr()),
                      f"hps_interface_solve(depth {d})")
        return Sp

    def panel_gemm(self, C, Sp):
        ne, n3, w = C.shape[1], C.shape[2], Sp.shape[2]
        Tp = self.empty((1, ne, w))
        _native.check(self.lib.hps_dgemm_batched(self.ctx, ne, w, n3, 1, 1.0, _native.ptr(C), n3, 0, _native.ptr(Sp),
                                                 w, 0, None, 0, 0.0, _native.ptr(Tp), w, 0, _native.stream_ptr()),
                      "hps_dgemm_batched(T panel)")
        return Tp

    def col_panel(self, M, c0, w):
        return M[:, :, c0:c0 + w].contiguous()

    def concat_cols(self, parts):
        return self.torch.cat(parts, dim=2).contiguous()

    def assemble(self, d, children, panels):
        dl = self.lay.depths[d]
        ne, m = dl.ne, dl.m
        P = self.torch.stack(panels).contiguous()  # (npanels, 1, ne, w)
        T = self.empty((1, ne, ne))
        _native.check(self.lib.hps_merge_assemble(self.ctx, 1, ne, m, _native.ptr(children), m * m, None,
                                                  _native.ptr(self.dl.maps[d]), _native.ptr(P), len(panels),
                                                  _native.ptr(T), _native.stream_ptr()), f"hps_merge_assemble({d})")
        return T

    def empty_int(self, shape):
        return self.torch.empty(shape, dtype=self.torch.int32, device=self.device)

    def read_failures(self, st):
        """(leaf cond array, [(depth, slot0, status value)]) of this rank, on the host."""
        cond = st.cond.cpu().numpy() if st.cond is not None else np.zeros(0)
        return cond, [(d, k, int(t.cpu().item())) for d, k, t in st.statuses]

    def solve_level(self, d, slot0, nslots, S, u, nrhs):
        dl = self.lay.depths[d]
        ldu = u.shape[1]
        Ie = self.dl.Ie[d][slot0:slot0 + nslots]
        start = int(self.lay.depth_off[d]) + slot0 * dl.n3
        _native.check(self.lib.hps_solve_level(self.ctx, nslots, dl.n3, dl.ne, _native.ptr(S), _native.ptr(Ie), start,
                                               _native.ptr(u), ldu, nrhs, _native.stream_ptr()), "hps_solve_level")

    def zeros(self, shape):
        return self.torch.zeros(shape, dtype=self.torch.float64, device=self.device)

    def stack2(self, a, b):
        return self.torch.cat([a, b], dim=0).contiguous()

    def status_word(self):
        return self.torch.full((1,), -1, dtype=self.torch.int32, device=self.device)


# ----------------------------------------------------------------------------------------------
# Orchestration
# ----------------------------------------------------------------------------------------------
@dataclass
class DistState:
    plan: SubtreePlan
    rank: int
    layout: object
    geom: object
    backend: object
    S_local: dict = field(default_factory=dict)   # depth -> S tensor for this rank's slots (d >= s)
    S_top: dict = field(default_factory=dict)     # depth -> S of the single owned box (d < s)
    subtree_T: object = None                       # DtN of this rank's depth-s box (before top merges)
    root_T: object = None                          # rank 0 only
    psi_groups: object = None
    T_leaf_groups: object = None
    leaf_group: np.ndarray = None                  # local leaf -> local group
    cond: object = None
    reps: np.ndarray = None                        # local leaf index of each group's first leaf
    statuses: list = field(default_factory=list)

    def owned_rows(self):
        """Global node ids whose solution this rank computes (its subtree's I_i ranges)."""
        lay, p = self.layout, self.plan
        rows = []
        for d in range(p.s, 2 * lay.L):
            lo, hi = p.local_slots(self.rank, d)
            n3 = lay.depths[d].n3
            rows.append(np.arange(lay.depth_off[d] + lo * n3, lay.depth_off[d] + hi * n3))
        for d in range(p.s):
            for k in p.top_boxes(self.rank, d):
                n3 = lay.depths[d].n3
                rows.append(np.arange(lay.depth_off[d] + k * n3, lay.depth_off[d] + (k + 1) * n3))
        return np.concatenate(rows) if rows else np.zeros(0, np.int64)


def _sample_local(coeffs, lay, geom, leaf_lo, leaf_hi):
    from .solver import COEFF_NAMES

    lc = lay.leaf_cells[leaf_lo:leaf_hi]
    xs = lay.xline[lc[:, 0]][:, None] + geom.grid_x[None, :]
    ys = lay.yline[lc[:, 1]][:, None] + geom.grid_y[None, :]
    fields = {}
    for name in COEFF_NAMES:
        f = getattr(coeffs, name)
        v = f(xs, ys) if callable(f) else float(f)
        if not np.all(np.isfinite(np.atleast_1d(v))):
            bad = np.argwhere(~np.isfinite(np.broadcast_to(v, xs.shape)))
            i, k = bad[0] if bad.size else (0, 0)
            raise ValueError(f"coefficient {name} is not finite at node ({xs[i, k]}, {ys[i, k]})")
        fields[name] = v if np.isscalar(v) else np.ascontiguousarray(np.broadcast_to(np.asarray(v, float), xs.shape))
    return fields


@dataclass
class LocalInputs:
    """This rank's sampled, grouped (and uploaded) leaf inputs."""

    fields: list
    scalars: list
    reps: np.ndarray
    gid: np.ndarray


def prepare_distributed(tree, coeffs, rank, world, backend):
    """Sample + group this rank's leaves and upload the group representatives (host work)."""
    from .solver import COEFF_NAMES, _group

    lay = layout_of(tree)
    plan = subtree_plan(lay.L, world)
    geom = LeafGeometry.get(lay.q, tree.leaf_width, tree.leaf_height)
    lo, hi = plan.local_slots(rank, 2 * lay.L)
    fields = _sample_local(coeffs, lay, geom, lo, hi)
    reps, gid = _group(fields, hi - lo)
    local_fields = [None if np.isscalar(fields[n]) else backend.upload(fields[n][reps]) for n in COEFF_NAMES]
    scalars = [float(fields[n]) if np.isscalar(fields[n]) else 0.0 for n in COEFF_NAMES]
    return LocalInputs(local_fields, scalars, reps, gid)


def _merge_flags(d, pivoted):
    return (_native.HPS_MERGE_PIVOTED if d in pivoted else 0) | \
        (_native.HPS_MERGE_PARENT_PIVOTED if d - 1 in pivoted else 0)


def top_groups(s):
    """The rank groups of the top merges (depths s-1 .. 0; group of parent k at depth d = ranks
    [k 2^(s-d), (k+1) 2^(s-d))), in the order every rank creates them."""
    out = []
    for d in range(s - 1, -1, -1):
        P = 1 << (s - d)
        out.extend(tuple(range(k * P, (k + 1) * P)) for k in range(1 << d))
    return out


def build_distributed(tree, coeffs, comm, backend, inputs=None, top_mode="panels", check=True, pivoted=()):
    """Subtree-parallel build. `comm` provides rank, world, send(tensor, dst), recv(tensor, src).
    `inputs` (from prepare_distributed) skips the host sampling/grouping. `top_mode` is "panels"
    (the top merges' solves and T GEMMs split in column panels over the parent's group) or "owner"
    (the parent's owner merges alone). With check=True every rank raises the reference's exception
    for the first failure in the reference's order (check_distributed), and depths whose fast
    interface inverse failed its residual check are rebuilt on the pivoted LU (`pivoted`)."""
    pivoted = frozenset(pivoted)
    lay = layout_of(tree)
    L = lay.L
    plan = subtree_plan(L, comm.world)
    rank, s = comm.rank, plan.s
    geom = LeafGeometry.get(lay.q, tree.leaf_width, tree.leaf_height)
    st = DistState(plan=plan, rank=rank, layout=lay, geom=geom, backend=backend)
    if inputs is None:
        inputs = prepare_distributed(tree, coeffs, rank, comm.world, backend)
    gid = inputs.gid
    Psi, Tleaf, cond = backend.leaf_stage(inputs.fields, inputs.scalars, int(inputs.reps.size))
    st.psi_groups, st.T_leaf_groups, st.leaf_group, st.cond = Psi, Tleaf, gid, cond
    st.reps = inputs.reps

    # ---- local merges, depths 2L-1 .. s (the parents of a local depth above s are local too, so
    # their status words exist one call early for the look-ahead inverse) ----
    child_T, child_idx = Tleaf, gid
    ahead_status = {}
    for d in range(2 * L - 1, s - 1, -1):
        a, b = plan.local_slots(rank, d)
        status = ahead_status.pop(d, None)
        if status is None:
            status = backend.status_word()
        st.statuses.append((d, a, status))
        pstatus = None
        if d - 1 >= s:
            pstatus = ahead_status[d - 1] = backend.status_word()
        S, T = backend.merge_level(d, b - a, child_T, child_idx, status, parent_status=pstatus, pivoted=pivoted)
        st.S_local[d] = S
        child_T, child_idx = T, None
    if s == 2 * L:  # one leaf per rank
        child_T = Tleaf[gid[0]:gid[0] + 1]
    st.subtree_T = child_T  # (1, ne_s, ne_s)

    # ---- top merges, depths s-1 .. 0. Child b's owner sends its DtN map to the
    # parent's owner (child a's owner), which forms and factors the interface system. "panels"
    # (default): every rank of the parent's group (2^(s-d) ranks) then solves a column panel of S and
    # forms the matching column panel of T = C S, so the dominant T GEMM (and the triangular solves)
    # run on all ranks instead of one; the owner assembles T = blkdiag + panels and keeps S for the
    # solve. "owner": the owner merges alone (hps_merge_level). Same per-element arithmetic. ----
    cur = child_T
    if top_mode == "panels" and hasattr(comm, "setup_groups"):  # every rank, same order: collective
        comm.setup_groups(top_groups(s))
    for d in range(s - 1, -1, -1):
        P = 1 << (s - d)  # ranks in the parent's group
        k = rank >> (s - d)
        owner = k << (s - d)
        span = P // 2
        dl = lay.depths[d]
        m = dl.m
        other = None
        if rank % span == 0:
            kc = rank // span
            if kc % 2 == 1:
                comm.send(cur, owner)
                cur = None
            else:
                other = backend.empty((1, m, m))
                comm.recv(other, owner + span)
        panels = top_mode == "panels" and dl.n3 >= 64 and dl.ne % P == 0 and (dl.ne // P) % 2 == 0
        if not panels:
            if rank == owner:
                status = backend.status_word()
                st.statuses.append((d, k, status))
                S, T = backend.merge_level(d, 1, backend.stack2(cur, other), None, status, pivoted=pivoted)
                st.S_top[d] = S
                cur = T
            continue
        n3, ne, w = dl.n3, dl.ne, dl.ne // P
        status = backend.status_word()
        st.statuses.append((d, k, status))
        group = tuple(range(owner, owner + P))
        if rank == owner:
            children = backend.stack2(cur, other)
            Xf, perm, R, C = backend.merge_interface(d, children, status, pivoted=pivoted)
            for r in range(1, P):
                comm.send(backend.col_panel(R, r * w, w), owner + r)
            Rp = backend.col_panel(R, 0, w)
        else:
            Xf, perm = backend.empty((1, n3, n3)), backend.empty_int((1, n3))
            C, Rp = backend.empty((1, ne, n3)), backend.empty((1, n3, w))
            comm.recv(Rp, owner)
        # the factored interface and C are the same for every rank of the group: one broadcast each
        # (NCCL pipelines it; the owner no longer sends them P - 1 times)
        for t in (Xf, perm, C):
            if hasattr(comm, "bcast"):
                comm.bcast(t, owner, group)
            elif rank == owner:
                for r in range(1, P):
                    comm.send(t, owner + r)
            else:
                comm.recv(t, owner)
        Sp = backend.interface_solve(d, Xf, perm, Rp, status, pivoted=pivoted)
        Tp = backend.panel_gemm(C, Sp)
        if rank == owner:
            Tps, Sps = [Tp], [Sp]
            for r in range(1, P):
                t, sp = backend.empty((1, ne, w)), backend.empty((1, n3, w))
                comm.recv(t, owner + r)
                comm.recv(sp, owner + r)
                Tps.append(t)
                Sps.append(sp)
            cur = backend.assemble(d, children, Tps)
            st.S_top[d] = backend.concat_cols(Sps)
        else:
            comm.send(Tp, owner)
            comm.send(Sp, owner)
            cur = None
    if rank == 0:
        st.root_T = cur
    if check:
        retry = check_distributed(st, comm) - pivoted
        if retry:
            return build_distributed(tree, coeffs, comm, backend, inputs, top_mode, check, pivoted | retry)
    return st


def check_distributed(st, comm):
    """Raise on every rank the exception the single-process build would raise: LeafResonanceError for
    the first resonant leaf group (smallest global leaf index of a bad group's first leaf), else
    MergeResonanceError for the first failing merge in the reference's order (deepest first,
    highest box index first; solver.py:235-239, 280-281). One host sync and a min-reduction.
    Returns the depths (on any rank) whose fast interface inverse failed its residual check."""
    from .errors import LeafResonanceError, MergeResonanceError
    from .solver import RESONANCE_COND

    lay, plan = st.layout, st.plan
    n_leaf = 1 << (2 * lay.L)
    cond, statuses = st.backend.read_failures(st)
    key, info = n_leaf + (1 << (2 * lay.L + 1)), None  # "no failure"
    bad = np.flatnonzero(cond > RESONANCE_COND)
    if bad.size:
        lo, _ = plan.local_slots(st.rank, 2 * lay.L)
        g = int(bad[0])
        leaf = lo + int(st.reps[g])
        key, info = leaf, float(cond[g])
    retry = {d for d, k, v in statuses if v >= _native.HPS_STATUS_PIVOT}
    if not bad.size:
        boxes = [(1 << d) - 1 + k + v for d, k, v in statuses if 0 <= v < _native.HPS_STATUS_PIVOT]
        if boxes:
            box = max(boxes)
            key = n_leaf + ((1 << (2 * lay.L + 1)) - 1 - box)
    keys = comm.allgather_obj((key, info, sorted(retry)))
    retry = set().union(*[set(k[2]) for k in keys])
    key, info = min(((k[0], k[1]) for k in keys), key=lambda x: x[0])
    if retry and key >= n_leaf:
        return retry  # rebuild first: a merge failure may be a consequence of the inaccurate inverse
    if key < n_leaf:
        raise LeafResonanceError(box=n_leaf - 1 + key, cond=info)
    if key < n_leaf + (1 << (2 * lay.L + 1)):
        box = (1 << (2 * lay.L + 1)) - 1 - (key - n_leaf)
        raise MergeResonanceError(box=box, detail="non-finite solution operator")
    return retry


def solve_distributed(st, F, comm):
    """Subtree-parallel batched solve. F: (|Gamma|, b) on rank 0 (ignored elsewhere), in root.I_e
    order. Returns this rank's u buffer (N x ldu); rows in st.owned_rows() plus the subtree's
    boundary are valid."""
    from .solver import rhs_ld

    be, lay, plan, rank = st.backend, st.layout, st.plan, st.rank
    L, s = lay.L, plan.s
    b = int(F.shape[1]) if F is not None and len(F.shape) > 1 else 1
    b = comm.bcast_int(b)
    ldu = rhs_ld(b)
    nrhs = b if b <= 8 else ldu
    u = be.zeros((lay.N, ldu))
    if rank == 0:
        Fm = F if len(F.shape) > 1 else F[:, None]
        be.scatter_rows(u, lay.root_I_e, Fm)
    # top depths: owners apply S, then hand child-b boundary values to child b's owner
    for d in range(s):
        for k in plan.top_boxes(rank, d):
            be.solve_level(d, k, 1, st.S_top[d], u, nrhs)
            kb = 2 * k + 1
            dst = plan.owner(d + 1, kb)
            if dst != rank:
                ids = lay.depths[d + 1].I_e[kb] if d + 1 < 2 * L else lay.leaf_I_e[kb]
                comm.send(be.gather_rows(u, ids), dst)
        # receive my subtree's (or my child-b box's) boundary values from the parent owner
        if rank % (1 << (s - d - 1)) == 0 and (rank >> (s - d - 1)) % 2 == 1:
            kb = rank >> (s - d - 1)
            ids = lay.depths[d + 1].I_e[kb] if d + 1 < 2 * L else lay.leaf_I_e[kb]
            buf = be.zeros((len(ids), ldu))
            comm.recv(buf, plan.owner(d, kb // 2))
            be.scatter_rows(u, ids, buf)
    for d in range(s, 2 * L):
        a, bb = plan.local_slots(rank, d)
        be.solve_level(d, a, bb - a, st.S_local[d], u, nrhs)
    return u


def gather_solution(st, u, comm, b):
    """Assemble the full (N, b) solution on rank 0 from the sharded buffers (others get None)."""
    be = st.backend
    rows = st.owned_rows()
    mine = be.gather_rows(u, rows)
    if comm.rank != 0:
        comm.send_obj(rows, 0)
        comm.send(mine, 0)
        return None
    out = be.zeros(u.shape)
    be.scatter_rows(out, st.layout.root_I_e, be.gather_rows(u, st.layout.root_I_e))
    be.scatter_rows(out, rows, mine)
    for src in range(1, comm.world):
        r = comm.recv_obj(src)
        buf = be.zeros((len(r), u.shape[1]))
        comm.recv(buf, src)
        be.scatter_rows(out, r, buf)
    return be.to_numpy(out)[:, :b]


class TorchComm:
    """torch.distributed transport (NCCL for device tensors, gloo for host tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._groups = {}

    def setup_groups(self, groups):
        """Create the process subgroups `groups` (tuples of ranks). Collective: every rank calls it
        with the same list in the same order (torch.distributed.new_group's rule)."""
        for g in groups:
            g = tuple(g)
            if g not in self._groups:
                self._groups[g] = self.group if len(g) == self.world else self.dist.new_group(list(g))

    def bcast(self, t, src, ranks):
        """Broadcast t from rank src to `ranks` (a group set up by setup_groups): one NCCL
        broadcast (pipelined over NVLink), so the source sends the data about once instead of once
        per receiver."""
        g = self._groups.get(tuple(ranks))
        if g is None:
            if self.rank == src:
                for r in ranks:
                    if r != src:
                        self.send(t, r)
            else:
                self.recv(t, src)
            return
        self.dist.broadcast(t, src, group=g)

    def send(self, t, dst):
        self.dist.send(t.contiguous(), dst, group=self.group)

    def recv(self, t, src):
        self.dist.recv(t, src, group=self.group)

    def bcast_int(self, v):
        obj = [v]
        self.dist.broadcast_object_list(obj, src=0, group=self.group)
        return int(obj[0])

    def send_obj(self, o, dst):
        self.dist.send_object_list([o], dst, group=self.group)

    def allgather_obj(self, o):
        out = [None] * self.world
        self.dist.all_gather_object(out, o, group=self.group)
        return out

    def recv_obj(self, src):
        obj = [None]
        self.dist.recv_object_list(obj, src, group=self.group)
        return obj[0]


class LocalComm:
    """In-process transport for `world` ranks run as threads of one process, sharing one device
    (the 2/4/8-way partition on one GPU, device-to-device copies in place of
    NCCL). `LocalComm.run(world, fn)` calls fn(comm) on every rank's thread and returns the results
    in rank order. Sends are device copies (the sender's tensor is cloned when sent)."""

    def __init__(self, rank, world, hub):
        self.rank, self.world, self._hub = rank, world, hub

    @staticmethod
    def run(world, fn):
        import queue
        import threading

        hub = {"q": {(a, b): queue.Queue() for a in range(world) for b in range(world)},
               "barrier": threading.Barrier(world), "slots": [None] * world}
        results, errors = [None] * world, [None] * world

        def body(r):
            try:
                results[r] = fn(LocalComm(r, world, hub))
            except BaseException as e:  # noqa: BLE001 -- re-raised on the caller's thread
                errors[r] = e
                hub["barrier"].abort()

        ths = [threading.Thread(target=body, args=(r,)) for r in range(world)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        for e in errors:
            if e is not None and not isinstance(e, threading.BrokenBarrierError):
                raise e
        for e in errors:
            if e is not None:
                raise e
        return results

    def send(self, t, dst):
        self._hub["q"][(self.rank, dst)].put(t.clone())

    def recv(self, t, src):
        t.copy_(self._hub["q"][(src, self.rank)].get(timeout=600))

    def send_obj(self, o, dst):
        self._hub["q"][(self.rank, dst)].put(o)

    def recv_obj(self, src):
        return self._hub["q"][(src, self.rank)].get(timeout=600)

    def allgather_obj(self, o):
        hub = self._hub
        hub["barrier"].wait()
        hub["slots"][self.rank] = o
        hub["barrier"].wait()
        out = list(hub["slots"])
        hub["barrier"].wait()
        return out

    def bcast_int(self, v):
        return int(self.allgather_obj(v)[0])

    def setup_groups(self, groups):
        pass

    def bcast(self, t, src, ranks):
        if self.rank == src:
            for r in ranks:
                if r != src:
                    self.send(t, r)
        else:
            self.recv(t, src)


def _cuda_backend_extras():
    """Row gather/scatter helpers on torch tensors (shared by the CUDA backend)."""

    def gather_rows(self, u, ids):
        idx = self.torch.as_tensor(np.asarray(ids, np.int64), device=u.device)
        return u.index_select(0, idx).contiguous()

    def scatter_rows(self, u, ids, vals):
        idx = self.torch.as_tensor(np.asarray(ids, np.int64), device=u.device)
        v = vals if hasattr(vals, "to") else self.torch.from_numpy(np.ascontiguousarray(vals))
        v = v.to(u.device, self.torch.float64)
        u[:, :v.shape[1]].index_copy_(0, idx, v)

    CudaBackend.gather_rows = gather_rows
    CudaBackend.scatter_rows = scatter_rows


_cuda_backend_extras()
