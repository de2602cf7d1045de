"""The C-ABI boundary (include/hps_b200.h) and loud failure without a GPU, CPU only."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1307_2665_b200 import _native
from paper_1307_2665_b200.errors import NativeError

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "hps_b200.h")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hps_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for sym in header_symbols():
        assert hasattr(lib, sym), sym
    assert lib.hps_version() >= 1
    assert isinstance(lib.hps_launch_count(), int)


def test_workspace_queries_are_host_only():
    lib = _native.load()
    ni, nb = 14 * 14, 60
    assert lib.hps_leaf_workspace_bytes(None, 16, 1) >= ni * (ni + nb + 1) * 8
    assert lib.hps_merge_workspace_bytes(4, 32, 128) >= 4 * (32 * 32 + 2 * 32 * 128) * 8


def test_context_calls_reject_a_null_context():
    lib = _native.load()
    assert lib.hps_ctx_get_option(None, _native.HPS_OPT_SPLITK) == -1
    assert lib.hps_ctx_set_option(None, _native.HPS_OPT_SPLITK, 0) == _native.HPS_ERR_ARG
    assert lib.hps_ctx_device(None) == -1
    assert lib.hps_ctx_destroy(None) == _native.HPS_OK
    st = lib.hps_dgemm_batched(None, 4, 4, 16, 1, 1.0, None, 16, 0, None, 4, 0, None, 0, 0.0, None, 4, 0, None)
    assert st == _native.HPS_ERR_ARG and "null hps_ctx_t" in _native.last_error()


def test_library_has_no_environment_knobs():
    """Settings live in the context (hps_ctx_set_option), not in getenv calls inside the library's
    sources (the static CUDA runtime it links reads its own variables)."""
    import glob
    csrc = os.path.join(os.path.dirname(_native.__file__), "csrc")
    for path in glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cuh")):
        assert "getenv(" not in open(path).read(), path


def test_no_cpu_fallback():
    """Without a device the product path raises; nothing silently computes on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1307_2665_b200 as P
    from paper_1307_2665_b200 import solver

    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 1, 16)
    with pytest.raises(NativeError):
        solver.build(tree, nodes, P.CoefficientField())


def test_nonfinite_coefficient_raises_valueerror_first():
    import paper_1307_2665_b200 as P
    from paper_1307_2665_b200 import solver

    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 1, 16)
    bad = P.CoefficientField(c=lambda x, y: np.where(x > 0.7, np.nan, 0.0))
    with pytest.raises(ValueError, match="coefficient c is not finite"):
        solver.build(tree, nodes, bad)


def test_pointer_guard_rejects_strided_views():
    import torch

    t = torch.zeros(4, 6, dtype=torch.float64).t()
    with pytest.raises(NativeError):
        _native.ptr(t)
    assert _native.ptr(None).value is None
