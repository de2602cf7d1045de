"""Generate golden vectors from the REFERENCE implementation (run in the build container, where
/root/reference exists): PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed, small):
  tree_small.npz        full layout of small trees (bit-exact gate)
  tree_hashes.json      sha256 of the layout arrays of larger trees (L = 4..7, q = 16)
  cfg{1..5}_L2.npz      leaf T / Psi / cond, leaf-pair S and T, root T, per-leaf L1 u for
                        seeded boundary data (b = 2), all from hpsolve.solver.build(...,
                        switch_threshold=None) and hpsolve.solver.solve
The boundary data and coefficient fields come from paper_1307_2665_b200.problems (the generators
of the five BASELINE configs), so both sides see identical inputs.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")

from hpsolve import grid, leafops, merge, solver  # noqa: E402  (the reference)
from paper_1307_2665_b200 import problems  # noqa: E402  (generators only)

AXIS = {"v": 0, "h": 1, "none": 2}


def tree_arrays(domain, L, q):
    t, n = grid.build_tree(grid.Rectangle(*domain), L, q)
    Ie = [b.I_e for b in t.boxes]
    Ii = [b.I_i if b.I_i is not None else np.zeros(0, np.intp) for b in t.boxes]
    return {
        "points": n.points, "on_vertical": n.on_vertical, "n_gamma": np.array(n.n_gamma),
        "cells": np.array([b.cells for b in t.boxes], np.int64),
        "axis": np.array([AXIS[b.split_axis] for b in t.boxes], np.int8),
        "parent": np.array([-1 if b.parent is None else b.parent for b in t.boxes], np.int64),
        "child_a": np.array([-1 if b.child_a is None else b.child_a for b in t.boxes], np.int64),
        "Ie_flat": np.concatenate(Ie).astype(np.int64), "Ie_len": np.array([len(x) for x in Ie], np.int64),
        "Ii_flat": np.concatenate(Ii).astype(np.int64), "Ii_len": np.array([len(x) for x in Ii], np.int64),
    }


def digest(arrs):
    h = hashlib.sha256()
    for k in sorted(arrs):
        a = np.ascontiguousarray(arrs[k])
        h.update(k.encode())
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def main():
    small = {}
    for tag, (dom, L, q) in {"u_L0_q5": ((0, 1, 0, 1), 0, 5), "u_L1_q16": ((0, 1, 0, 1), 1, 16),
                             "u_L2_q16": ((0, 1, 0, 1), 2, 16), "odd_L2_q7": ((-0.3, 2.1, 0.7, 1.9), 2, 7),
                             "u_L3_q16": ((0, 1, 0, 1), 3, 16), "u_L2_q21": ((0, 1, 0, 1), 2, 21)}.items():
        for k, v in tree_arrays(dom, L, q).items():
            small[f"{tag}__{k}"] = v
    np.savez_compressed(os.path.join(HERE, "tree_small.npz"), **small)
    hashes = {f"L{L}_q16": digest(tree_arrays((0, 1, 0, 1), L, 16)) for L in (4, 5, 6, 7)}
    with open(os.path.join(HERE, "tree_hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1)

    L = 2
    for cfg in (1, 2, 3, 4, 5):
        co = problems.coefficients(cfg)
        ref = leafops.CoefficientField(**{n: getattr(co, n) for n in ("c11", "c12", "c22", "c1", "c2", "c")})
        t, n = grid.build_tree(grid.Rectangle(0, 1, 0, 1), L, 16)
        geom = leafops.LeafGeometry.get(16, t.leaf_width, t.leaf_height)
        psi, Tl, ng = solver._leaf_stage(t, n, ref, geom)
        leaves = t.leaves()
        # group representatives in first-occurrence order, as the reference dedups them
        seen, reps = {}, []
        for b in leaves:
            key = psi[b.index].__array_interface__["data"][0]
            if key not in seen:
                seen[key] = len(reps)
                reps.append(b.index)
        out = {"leaf_T": np.stack([Tl[i] for i in reps[:4]]), "psi": np.stack([psi[i] for i in reps[:2]]),
               "rep_leaf_index": np.array(reps, np.int64),
               "leaf_group": np.array([seen[psi[b.index].__array_interface__["data"][0]] for b in leaves], np.int64)}
        # replay the dense merges, keeping the leaf-pair level S/T (well-conditioned) and the root
        Tstore = dict(Tl)
        for box in reversed(t.boxes):
            if box.is_leaf:
                continue
            sp = merge.split_indices(box, t.boxes[box.child_a], t.boxes[box.child_b])
            S, T = merge.merge_dtn(Tstore.pop(box.child_a), Tstore.pop(box.child_b), sp)
            Tstore[box.index] = T
            if box.index in (7, 8):  # leaf-pair merges at depth 2L-1 (X nonsingular there)
                out[f"S_box{box.index}"] = S
                out[f"T_box{box.index}"] = T
        st = solver.build(t, n, ref, switch_threshold=None)
        out["root_T"] = st.root_T.dense
        assert np.array_equal(out["root_T"], Tstore[0])
        F = problems.boundary_data(cfg, n.points[t.root.I_e], seed=11, batch=2)
        out["F"] = F
        U = np.stack([solver.solve(st, F[:, j]) for j in range(F.shape[1])], axis=1)
        out["L1u"] = np.stack([geom.L1 @ U[b.I_e] for b in leaves])
        # the probe condition estimates of every group
        A = np.stack([leafops.build_local_operator(ref, b.rect, 16) for b in (t.boxes[i] for i in reps)])
        _, conds = leafops.interior_solve_batch(geom, A)
        out["cond"] = conds
        np.savez_compressed(os.path.join(HERE, f"cfg{cfg}_L{L}.npz"), **out)
        print(cfg, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
