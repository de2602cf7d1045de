"""Bit-exact tree / node layout (bit-exact gate), CPU only.

The product's closed-form layout (paper_1307_2665_b200.grid) is compared against the golden
vectors produced by the reference's own build_tree (tests/golden/make_golden.py) and against the
oracle restatement."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import hps_oracle as O
from paper_1307_2665_b200 import grid as G

from _util import GOLDEN, golden_tree

AXIS = {"v": 0, "h": 1, "none": 2}
SMALL = {"u_L0_q5": ((0, 1, 0, 1), 0, 5), "u_L1_q16": ((0, 1, 0, 1), 1, 16), "u_L2_q16": ((0, 1, 0, 1), 2, 16),
         "odd_L2_q7": ((-0.3, 2.1, 0.7, 1.9), 2, 7), "u_L3_q16": ((0, 1, 0, 1), 3, 16),
         "u_L2_q21": ((0, 1, 0, 1), 2, 21)}


def product_arrays(dom, L, q):
    t, n = G.build_tree(G.Rectangle(*dom), L, q)
    Ie = [t.boxes[i].I_e for i in range(t.n_boxes)]
    Ii = [t.boxes[i].I_i if t.boxes[i].I_i is not None else np.zeros(0, np.intp) for i in range(t.n_boxes)]
    bx = [t.boxes[i] for i in range(t.n_boxes)]
    return {
        "points": n.points, "on_vertical": n.on_vertical, "n_gamma": np.array(n.n_gamma),
        "cells": np.array([b.cells for b in bx], np.int64),
        "axis": np.array([AXIS[b.split_axis] for b in bx], np.int8),
        "parent": np.array([-1 if b.parent is None else b.parent for b in bx], np.int64),
        "child_a": np.array([-1 if b.child_a is None else b.child_a for b in bx], np.int64),
        "Ie_flat": np.concatenate(Ie).astype(np.int64), "Ie_len": np.array([len(x) for x in Ie], np.int64),
        "Ii_flat": np.concatenate(Ii).astype(np.int64), "Ii_len": np.array([len(x) for x in Ii], np.int64),
    }


@pytest.mark.parametrize("tag", sorted(SMALL))
def test_layout_matches_reference_golden(tag):
    ref = golden_tree(tag)
    got = product_arrays(*SMALL[tag])
    assert set(ref) == set(got)
    for k in ref:
        assert ref[k].shape == got[k].shape, k
        assert np.array_equal(ref[k], got[k]), k  # bitwise, including the fp64 points


@pytest.mark.parametrize("L", [4, 5, 6, 7])
def test_layout_hash_matches_reference(L):
    with open(os.path.join(GOLDEN, "tree_hashes.json")) as f:
        want = json.load(f)[f"L{L}_q16"]
    arrs = product_arrays((0, 1, 0, 1), L, 16)
    h = hashlib.sha256()
    for k in sorted(arrs):
        a = np.ascontiguousarray(arrs[k])
        h.update(k.encode())
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    assert h.hexdigest() == want


@pytest.mark.parametrize("dom,L,q", [((0, 1, 0, 1), 3, 4), ((2.0, 3.5, -1.0, 0.25), 3, 9), ((0, 1, 0, 1), 4, 16)])
def test_layout_matches_oracle(dom, L, q):
    t, n = G.build_tree(G.Rectangle(*dom), L, q)
    o = O.build_tree(dom, L, q)
    assert np.array_equal(n.points, o.points) and np.array_equal(n.on_vertical, o.on_vertical)
    for i in range(o.n_boxes):
        assert np.array_equal(t.boxes[i].I_e, o.I_e[i])
        if o.child_a[i] >= 0:
            assert np.array_equal(t.boxes[i].I_i, o.I_i[i])


def test_spec_counts():
    # SPEC.md:83-85 and the node-count identity SPEC.md:99
    t, n = G.build_tree(G.Rectangle(0, 1, 0, 1), 2, 21)
    assert t.n_boxes == 31 and len(t.leaves()) == 16 and n.N == 840
    assert G.build_tree(G.Rectangle(0, 1, 0, 1), 0, 5)[1].N == 20
    lay = G.TreeLayout(G.Rectangle(0, 1, 0, 1), 6, 21)
    assert lay.N == 174720
    for L in range(0, 7):
        assert G.TreeLayout(G.Rectangle(0, 1, 0, 1), L, 16).N == 2 ** (2 * L + 1) * 16 + 2 ** (L + 1) * 16


def test_spec_nodes_and_interp():
    assert np.allclose(G.gauss_nodes(2), [-0.57735026919, 0.57735026919], atol=1e-11)
    assert np.array_equal(G.gauss_nodes(1), [0.0])
    assert np.allclose(G.cheb_nodes(5), [-1, -np.sqrt(2) / 2, 0, np.sqrt(2) / 2, 1], atol=1e-15)
    g = G.gauss_nodes(21)
    assert np.allclose(g, -g[::-1], atol=1e-14) and np.abs(g).max() < 1
    src = G.cheb_nodes(9, (0.0, 2.0))
    dst = np.linspace(0, 2, 13)
    M = G.interp_matrix(src, dst)
    for deg in range(9):  # exact for degree <= p-1
        assert np.allclose(M @ src ** deg, dst ** deg, atol=1e-11 * 2 ** deg)
    with pytest.raises(ValueError):
        G.interp_matrix([0.0, 0.0], [1.0])
    with pytest.raises(ValueError):
        G.build_tree(G.Rectangle(0, 1, 0, 1), -1, 16)
    with pytest.raises(ValueError):
        G.build_tree(G.Rectangle(0, 1, 0, 1), 2, 1)
    with pytest.raises(ValueError):
        G.Rectangle(1, 0, 0, 1)


@pytest.mark.parametrize("L", [2, 3, 5])
def test_split_maps_uniform_and_consistent(L):
    """Every parent at a depth shares one split map (what lets a depth run as one batch)."""
    lay = G.TreeLayout(G.Rectangle(0, 1, 0, 1), L, 16)
    t = G.BoxTree(lay)
    for d, dl in enumerate(lay.depths):
        assert dl.ne == dl.j1a.size + dl.j2b.size and dl.m == dl.ne // 2 + dl.n3
        n3, ne = O.depth_sizes(L, 16, d)
        assert (dl.n3, dl.ne) == (n3, ne)
        for k in (0, dl.n_boxes - 1):
            box = (1 << d) - 1 + k
            j1a, j2b, j3a, j3b = O.split_indices(t.boxes[2 * box + 1].I_e, t.boxes[2 * box + 2].I_e,
                                                 t.boxes[box].I_i)
            assert np.array_equal(j1a, dl.j1a) and np.array_equal(j2b, dl.j2b)
            assert np.array_equal(j3a, dl.j3a) and np.array_equal(j3b, dl.j3b)


def test_box_accessors():
    t, n = G.build_tree(G.Rectangle(0, 1, 0, 1), 2, 16)
    leaf = t.leaf_at(1, 2)
    assert leaf.cells[:2] == (1, 2) and leaf.is_leaf
    assert t.root.index == 0 and not t.root.is_leaf
    assert len(t.parents()) == 15
    assert t.boxes[-1].index == t.n_boxes - 1


@pytest.mark.parametrize("dom,L,q", [((0, 1, 0, 1), 0, 16), ((0, 1, 0, 1), 1, 16), ((0, 1, 0, 1), 5, 16),
                                     ((-0.3, 1.7, 0.25, 0.75), 3, 7), ((0, 2, 0, 1), 4, 21)])
def test_native_layout_builder_is_identical(dom, L, q, monkeypatch):
    # csrc/tree.cu (hps_tree_layout) against the numpy closed forms: every
    # array bit for bit (coordinates as bit patterns), every per-depth map and I_e list
    from paper_1307_2665_b200.grid import TreeLayout
    monkeypatch.setenv("HPS_NATIVE_LAYOUT", "1")
    a = TreeLayout(G.Rectangle(*dom), L, q)
    monkeypatch.setenv("HPS_NATIVE_LAYOUT", "0")
    b = TreeLayout(G.Rectangle(*dom), L, q)
    for k in ("n_gamma", "N", "n3s", "depth_off"):
        assert getattr(a, k) == getattr(b, k), k
    for k in ("xline", "yline", "points", "on_vertical", "leaf_cells", "leaf_I_e", "root_I_e"):
        x, y = getattr(a, k), getattr(b, k)
        assert x.shape == y.shape and x.dtype == y.dtype, k
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), k
    assert len(a.depths) == len(b.depths) == 2 * L
    for da, db in zip(a.depths, b.depths):
        for k in ("depth", "axis", "n3", "ne", "m"):
            assert getattr(da, k) == getattr(db, k), k
        for k in ("j1a", "j2b", "j3a", "j3b", "I_e", "Ii_start"):
            x, y = getattr(da, k), getattr(db, k)
            assert x.dtype == y.dtype and np.array_equal(x, y), (da.depth, k)
