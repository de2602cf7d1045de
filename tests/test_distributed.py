"""Multi-rank subtree build/solve over gloo on CPU, world_size 2 and 4.

paper_1307_2665_b200.parallel runs its orchestration unchanged. That covers the ownership plan,
the point-to-point moves of subtree-root DtN maps for the top merges, the top-down scatter of
interface data and the sharded output. The per-rank compute is a numpy backend defined here, so
the exchange logic can run without GPUs. Results are compared with the single-process oracle on
null-mode-invariant quantities.
"""
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1307_2665_b200 as P
from oracle import hps_oracle as O
from paper_1307_2665_b200 import parallel, problems
from paper_1307_2665_b200.grid import layout_of

from _util import coeff_dict, rel


class NumpyBackend:
    """CPU stand-in for CudaBackend with the same interface (torch CPU tensors for transport)."""

    def __init__(self, tree):
        self.lay = layout_of(tree)
        self.geom = O.Geometry(self.lay.q, tree.leaf_width, tree.leaf_height)

    def empty(self, shape):
        return torch.zeros(shape, dtype=torch.float64)

    zeros = empty

    def to_numpy(self, t):
        return t.numpy()

    def stack2(self, a, b):
        return torch.cat([a, b], 0).contiguous()

    def status_word(self):
        return torch.full((1,), -1, dtype=torch.int32)

    def upload(self, a):
        return a

    def leaf_stage(self, fields_local, scalars, ngroups):
        fields = {n: (scalars[i] if fields_local[i] is None else np.asarray(fields_local[i]))
                  for i, n in enumerate(O.COEFF_NAMES)}
        Psi, T, cond = O.leaf_operators(self.geom, fields, np.arange(ngroups))
        return torch.from_numpy(Psi), torch.from_numpy(T), torch.from_numpy(cond)

    def merge_level(self, d, nbatch, child_T, child_idx, status, parent_status=None, pivoted=()):
        dl = self.lay.depths[d]
        Tc = child_T.numpy()
        S, T = [], []
        for b in range(nbatch):
            ia, ib = (2 * b, 2 * b + 1) if child_idx is None else (child_idx[2 * b], child_idx[2 * b + 1])
            s_, t_ = O.merge_dtn(Tc[ia], Tc[ib], dl.j1a, dl.j2b, dl.j3a, dl.j3b)
            S.append(s_)
            T.append(t_)
        return torch.from_numpy(np.stack(S)), torch.from_numpy(np.stack(T))

    # split merge of the distributed top depths (the CUDA backend's hps_merge_interface & co.)
    def merge_interface(self, d, children, status, pivoted=()):
        dl = self.lay.depths[d]
        Ta, Tb = children[0].numpy(), children[1].numpy()
        X = Ta[np.ix_(dl.j3a, dl.j3a)] - Tb[np.ix_(dl.j3b, dl.j3b)]
        R = np.concatenate([-Ta[np.ix_(dl.j3a, dl.j1a)], Tb[np.ix_(dl.j3b, dl.j2b)]], axis=1)
        C = np.concatenate([Ta[np.ix_(dl.j1a, dl.j3a)], Tb[np.ix_(dl.j2b, dl.j3b)]])
        perm = np.arange(dl.n3, dtype=np.int32)
        return tuple(torch.from_numpy(np.ascontiguousarray(a)[None]) for a in (X, perm, R, C))

    def interface_solve(self, d, Xf, perm, Rp, status, pivoted=()):
        import scipy.linalg as sla
        X = Xf[0].numpy()[perm[0].numpy()]
        return torch.from_numpy(sla.lu_solve(sla.lu_factor(X), Rp[0].numpy()[perm[0].numpy()])[None])

    def panel_gemm(self, C, Sp):
        return torch.from_numpy((C[0].numpy() @ Sp[0].numpy())[None])

    def col_panel(self, M, c0, w):
        return M[:, :, c0:c0 + w].contiguous()

    def concat_cols(self, parts):
        return torch.cat(parts, dim=2).contiguous()

    def assemble(self, d, children, panels):
        dl = self.lay.depths[d]
        Ta, Tb = children[0].numpy(), children[1].numpy()
        T = np.concatenate([p[0].numpy() for p in panels], axis=1)
        n1 = dl.j1a.size
        T[:n1, :n1] += Ta[np.ix_(dl.j1a, dl.j1a)]
        T[n1:, n1:] += Tb[np.ix_(dl.j2b, dl.j2b)]
        return torch.from_numpy(T[None])

    def empty_int(self, shape):
        return torch.zeros(shape, dtype=torch.int32)

    def read_failures(self, st):
        return st.cond.numpy(), [(d, k, int(t.item())) for d, k, t in st.statuses]

    def solve_level(self, d, slot0, nslots, S, u, nrhs):
        dl = self.lay.depths[d]
        un = u.numpy()
        for j in range(nslots):
            k = slot0 + j
            start = self.lay.depth_off[d] + k * dl.n3
            un[start:start + dl.n3, :nrhs] = S[j].numpy() @ un[dl.I_e[k], :nrhs]

    def gather_rows(self, u, ids):
        return torch.from_numpy(np.ascontiguousarray(u.numpy()[np.asarray(ids)]))

    def scatter_rows(self, u, ids, vals):
        v = vals.numpy() if hasattr(vals, "numpy") else np.asarray(vals)
        u.numpy()[np.asarray(ids), :v.shape[1]] = v


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, L, b, out, top_mode="panels"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tree, nodes = P.build_tree(P.Rectangle(0.0, 1.0, 0.0, 1.0), L, 16)
        be = NumpyBackend(tree)
        comm = parallel.TorchComm()
        st = parallel.build_distributed(tree, problems.coefficients(cfg), comm, be, top_mode=top_mode)
        F = None
        if rank == 0:
            F = torch.from_numpy(problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=5, batch=b))
        u = parallel.solve_distributed(st, F, comm)
        full = parallel.gather_solution(st, u, comm, b)
        if rank == 0:
            with open(out, "wb") as f:
                pickle.dump({"root_T": st.root_T[0].numpy(), "u": full,
                             "F": F.numpy(), "owned": st.owned_rows()}, f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg,L,top_mode", [(2, 2, 2, "panels"), (4, 2, 2, "panels"), (4, 3, 2, "owner"),
                                                  (2, 5, 1, "panels"), (8, 2, 2, "panels"), (8, 4, 2, "owner"),
                                                  (4, 5, 3, "panels")])
def test_subtree_build_and_solve_match_single_process(world, cfg, L, top_mode):
    """World 8 is the 2 x 4 subtree split of SURVEY.md §8e (boxes 7..14)."""
    b = 3
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "r0.pkl")
        mp.spawn(_worker, args=(world, _free_port(), cfg, L, b, out, top_mode), nprocs=world, join=True)
        with open(out, "rb") as f:
            res = pickle.load(f)
    ot = O.build_tree((0, 1, 0, 1), L, 16)
    ost = O.build(ot, coeff_dict(problems.coefficients(cfg)))
    tol = 1e-10 if cfg != 3 else 1e-8
    assert rel(res["root_T"], ost.root_T) < tol
    uo = O.solve(ost, res["F"])
    assert rel(O.leaf_cheb_boundary(ost, res["u"]), O.leaf_cheb_boundary(ost, uo)) < tol


def test_subtree_plan():
    p = parallel.subtree_plan(3, 8)
    assert p.s == 3
    assert [p.owner(3, k) for k in range(8)] == list(range(8))
    assert [p.owner(2, k) for k in range(4)] == [0, 2, 4, 6]
    assert [p.owner(1, k) for k in range(2)] == [0, 4]
    assert p.owner(0, 0) == 0
    assert p.local_slots(5, 5) == (20, 24)
    assert p.top_boxes(4, 1) == [1] and p.top_boxes(2, 1) == [] and p.top_boxes(6, 2) == [3]
    with pytest.raises(P.ConfigError):
        parallel.subtree_plan(3, 6)
    with pytest.raises(P.ConfigError):
        parallel.subtree_plan(1, 16)
    # 8 ranks on L=9: depth-3 boxes 7..14 form a 4 (x) by 2 (y) grid
    lay = P.grid.TreeLayout(P.Rectangle(0, 1, 0, 1), 3, 16)
    ix, iy, nx, ny = lay.cells_at(3)
    assert (nx, ny) == (2, 4) and sorted(set(ix.tolist())) == [0, 2, 4, 6] and sorted(set(iy.tolist())) == [0, 4]


def _fail_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tree, nodes = P.build_tree(P.Rectangle(0.0, 1.0, 0.0, 1.0), 2, 16)
        be = NumpyBackend(tree)
        comm = parallel.TorchComm()
        st = parallel.build_distributed(tree, problems.coefficients(2), comm, be, check=False)
        got = []
        # a failing merge on rank 1's subtree (depth 3, its first local slot) and at the root (rank 0)
        st.statuses = [(d, k, torch.full((1,), 0 if (rank == 1 and d == 3) or (rank == 0 and d == 0) else -1,
                                         dtype=torch.int32)) for d, k, _ in st.statuses]
        try:
            parallel.check_distributed(st, comm)
        except P.MergeResonanceError as e:
            got.append(("merge", e.box))
        # a resonant leaf group on rank 1 takes precedence over any merge failure
        st.cond = st.cond.clone()
        if rank == 1:
            st.cond[0] = 1e20
        try:
            parallel.check_distributed(st, comm)
        except P.LeafResonanceError as e:
            got.append(("leaf", e.box))
        with open(out + f".{rank}", "wb") as f:
            pickle.dump(got, f)
    finally:
        dist.destroy_process_group()


def test_distributed_failures_raise_the_reference_exception_on_every_rank():
    """the multi-GPU build reads every rank's leaf cond and merge status words and raises
    the first failure in the reference's order (leaves first, then the deepest, highest box)."""
    world = 2
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "f")
        mp.spawn(_fail_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = [pickle.load(open(out + f".{r}", "rb")) for r in range(world)]
    plan = parallel.subtree_plan(2, world)
    lo, _ = plan.local_slots(1, 3)
    merge_box = (1 << 3) - 1 + lo  # rank 1's first depth-3 box (deeper, higher index than the root)
    leaf_lo, _ = plan.local_slots(1, 4)
    leaf_box = (1 << 4) - 1 + leaf_lo  # rank 1's first leaf (its group 0 representative)
    assert res[0] == res[1] == [("merge", merge_box), ("leaf", leaf_box)]
