"""Pin the oracle restatement to the reference's own outputs (golden vectors), CPU only."""
import numpy as np
import pytest

from oracle import hps_oracle as O
from paper_1307_2665_b200 import problems

from _util import coeff_dict, golden, rel


@pytest.fixture(scope="module", params=[1, 2, 3, 4, 5])
def case(request):
    cfg = request.param
    g = golden(f"cfg{cfg}_L2.npz")
    tree = O.build_tree((0, 1, 0, 1), 2, 16)
    st = O.build(tree, coeff_dict(problems.coefficients(cfg)), keep_T=True)
    return cfg, g, st


def test_leaf_operators(case):
    cfg, g, st = case
    k = g["leaf_T"].shape[0]
    assert rel(st.T_groups[:k], g["leaf_T"]) < 1e-13
    assert rel(st.psi_groups[:g["psi"].shape[0]], g["psi"]) < 1e-13
    assert rel(st.cond, g["cond"]) < 1e-12
    first = (1 << 4) - 1
    assert np.array_equal(np.array([st.tree.leaves[i] for i in st.reps]), g["rep_leaf_index"])
    assert np.array_equal(st.gid, g["leaf_group"])
    assert first == st.tree.leaves[0]


def test_merged_operators(case):
    cfg, g, st = case
    tol = 1e-13 if cfg in (1, 2, 5) else 1e-9
    for box in (7, 8):  # leaf-pair level: X nonsingular, so S is reproducible too
        assert rel(st.T[box], g[f"T_box{box}"]) < tol
        assert rel(st.S[box], g[f"S_box{box}"]) < tol
    assert rel(st.root_T, g["root_T"]) < tol


def test_solution_invariant(case):
    cfg, g, st = case
    u = O.solve(st, g["F"])
    tol = 1e-10 if cfg in (1, 2, 5) else 1e-8
    assert rel(O.leaf_cheb_boundary(st, u), g["L1u"]) < tol


def test_flop_model():
    # SURVEY.md §8a a9 / §8d totals
    assert abs(O.merge_flops(4, 16) - 1.95e9) / 1.95e9 < 0.01
    assert abs(O.merge_flops(6, 16) - 1.31e11) / 1.31e11 < 0.01
    assert abs(O.leaf_flops(16) - 1.170e7) / 1.17e7 < 0.01
    assert abs(O.solve_flops(6, 16, 64) - 5.64e9) / 5.64e9 < 0.01
