"""ctypes binding of libhps_b200.so (the C ABI declared in include/hps_b200.h).

There is no fallback. If the library is missing or no sm_100 device is visible, every entry point
raises. The product path never computes on the CPU.
"""

from __future__ import annotations

import ctypes
import os

from .errors import NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPS_LIB") or os.path.join(_HERE, "libhps_b200.so")

HPS_OK = 0
HPS_ERR_LEAF_RESONANCE = 1
HPS_ERR_MERGE_RESONANCE = 2
HPS_ERR_CUDA = 3
HPS_ERR_NCCL = 4
HPS_ERR_ARG = 5

#: every symbol include/hps_b200.h declares (tests check the .so exports all of them)
EXPORTS = ("hps_ctx_create", "hps_ctx_destroy", "hps_ctx_set_option", "hps_ctx_get_option", "hps_ctx_device",
           "hps_last_error", "hps_version", "hps_device_check", "hps_launch_count", "hps_leaf_workspace_bytes",
           "hps_leaf_stage", "hps_merge_workspace_bytes", "hps_merge_level", "hps_solve_level",
           "hps_dgemm_batched", "hps_inverse_workspace_bytes", "hps_inverse_batched", "hps_leaf_hash",
           "hps_leaf_verify", "hps_leaf_fields", "hps_eval_points", "hps_gauge_sides", "hps_gauge_gather",
           "hps_merge_level_ahead", "hps_tree_sizes", "hps_tree_layout", "hps_lu_workspace_bytes",
           "hps_lu_solve_batched", "hps_merge_interface", "hps_interface_solve", "hps_merge_assemble",
           "hps_i8gemm_mod")

HPS_OPT_SPLITK = 0
HPS_OPT_GEMM_GROUP_M = 1
HPS_OPT_INV_FORK = 2
HPS_OPT_LEAF_CTAS_PER_SM = 3
HPS_OPT_LEAF_FREE_SMS = 4
HPS_OPT_PROFILE_AHEAD = 5
HPS_OPT_EMU_SLICES = 6
HPS_OPT_EMU_MIN_WORK = 7
HPS_OPT_EMU_MIN_K = 8
HPS_OPT_EMU_MODULI = 9
HPS_OPT_EMU_SCRATCH_MB = 10
HPS_OPT_EMU_ENGINE = 11
HPS_OPT_EMU_TILE_GROUP = 12
HPS_OPT_EMU_SOLVE = 13
HPS_OPT_EMU_SPLIT = 14

HPS_MERGE_PIVOTED = 1
HPS_MERGE_PARENT_PIVOTED = 2
HPS_STATUS_PIVOT = 1 << 24

_lib = None

c_dp = ctypes.c_void_p
c_ll = ctypes.c_longlong
c_int = ctypes.c_int
c_sz = ctypes.c_size_t
c_d = ctypes.c_double


def load():
    """Load the shared library (no device work). Raises ImportError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() or csrc/build.sh; "
                          "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    lib.hps_last_error.restype = ctypes.c_char_p
    lib.hps_version.restype = c_int
    lib.hps_launch_count.restype = c_ll
    pll = ctypes.POINTER(c_ll)
    lib.hps_tree_sizes.argtypes = [c_int, c_int, pll, pll, pll]
    lib.hps_tree_sizes.restype = c_ll
    lib.hps_tree_layout.argtypes = [c_int, c_int, c_d, c_d, c_d, c_d, ctypes.POINTER(c_d), ctypes.POINTER(c_d),
                                    ctypes.POINTER(ctypes.c_ubyte), pll, pll, ctypes.POINTER(pll),
                                    ctypes.POINTER(pll)]
    lib.hps_tree_layout.restype = c_int
    lib.hps_ctx_create.argtypes = [c_int, ctypes.POINTER(c_dp)]
    lib.hps_ctx_create.restype = c_int
    lib.hps_ctx_destroy.argtypes = [c_dp]
    lib.hps_ctx_destroy.restype = c_int
    lib.hps_ctx_set_option.argtypes = [c_dp, c_int, c_ll]
    lib.hps_ctx_set_option.restype = c_int
    lib.hps_ctx_get_option.argtypes = [c_dp, c_int]
    lib.hps_ctx_get_option.restype = c_ll
    lib.hps_ctx_device.argtypes = [c_dp]
    lib.hps_ctx_device.restype = c_int
    lib.hps_device_check.argtypes = [ctypes.POINTER(c_int)] * 3
    lib.hps_device_check.restype = c_int
    lib.hps_leaf_workspace_bytes.argtypes = [c_dp, c_int, c_int]
    lib.hps_leaf_workspace_bytes.restype = c_sz
    lib.hps_leaf_stage.argtypes = [c_dp, c_int, c_int, ctypes.POINTER(c_dp), ctypes.POINTER(c_d), c_dp, c_dp, c_d,
                                   c_dp, c_dp, c_dp, c_dp, c_sz, c_dp]
    lib.hps_leaf_stage.restype = c_int
    lib.hps_merge_workspace_bytes.argtypes = [c_int, c_int, c_int]
    lib.hps_merge_workspace_bytes.restype = c_sz
    lib.hps_merge_level.argtypes = [c_dp, c_int, c_int, c_int, c_int, c_int, c_dp, c_ll, c_dp, c_dp, c_dp, c_dp, c_dp,
                                    c_dp, c_sz, c_dp, c_int, c_dp]
    lib.hps_merge_level.restype = c_int
    lib.hps_merge_level_ahead.argtypes = [c_dp, c_int, c_int, c_int, c_int, c_int, c_dp, c_ll, c_dp, c_dp, c_dp, c_dp, c_dp,
                                          c_dp, c_sz, c_dp, c_int, c_int, c_dp, c_int, c_int, c_dp, c_dp, c_sz, c_dp,
                                          c_int, c_int, c_dp]
    lib.hps_merge_level_ahead.restype = c_int
    lib.hps_debug_ahead_times.argtypes = [c_dp, c_int, ctypes.POINTER(ctypes.c_float)]
    lib.hps_debug_ahead_times.restype = c_int
    lib.hps_debug_ahead_depth.argtypes = [c_dp, c_int]
    lib.hps_debug_ahead_depth.restype = None
    lib.hps_solve_level.argtypes = [c_dp, c_int, c_int, c_int, c_dp, c_dp, c_ll, c_dp, c_int, c_int, c_dp]
    lib.hps_solve_level.restype = c_int
    lib.hps_dgemm_batched.argtypes = [c_dp, c_int, c_int, c_int, c_int, c_d, c_dp, c_ll, c_ll, c_dp, c_ll, c_ll, c_dp,
                                      c_ll, c_d, c_dp, c_ll, c_ll, c_dp]
    lib.hps_dgemm_batched.restype = c_int
    lib.hps_i8gemm_mod.argtypes = [c_dp, c_dp, c_dp, c_dp, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                   ctypes.POINTER(c_int), c_int, c_int, c_dp]
    lib.hps_i8gemm_mod.restype = c_int
    lib.hps_inverse_workspace_bytes.argtypes = [c_int, c_int]
    lib.hps_inverse_workspace_bytes.restype = c_sz
    lib.hps_inverse_batched.argtypes = [c_dp, c_int, c_int, c_dp, c_ll, c_ll, c_dp, c_sz, c_dp, c_dp]
    lib.hps_inverse_batched.restype = c_int
    lib.hps_lu_workspace_bytes.argtypes = [c_int, c_int]
    lib.hps_lu_workspace_bytes.restype = c_sz
    lib.hps_lu_solve_batched.argtypes = [c_dp, c_int, c_int, c_int, c_dp, c_dp, c_dp, c_dp, c_dp, c_sz, c_dp, c_dp]
    lib.hps_lu_solve_batched.restype = c_int
    lib.hps_merge_interface.argtypes = [c_dp, c_int, c_int, c_int, c_int, c_int, c_dp, c_ll, c_dp, c_dp, c_dp, c_dp,
                                        c_dp, c_dp, c_dp, c_dp, c_sz, c_dp, c_int, c_int, c_dp]
    lib.hps_merge_interface.restype = c_int
    lib.hps_interface_solve.argtypes = [c_dp, c_int, c_int, c_int, c_dp, c_dp, c_dp, c_dp, c_dp, c_int, c_int, c_dp]
    lib.hps_interface_solve.restype = c_int
    lib.hps_merge_assemble.argtypes = [c_dp, c_int, c_int, c_int, c_dp, c_ll, c_dp, c_dp, c_dp, c_int, c_dp, c_dp]
    lib.hps_merge_assemble.restype = c_int
    lib.hps_leaf_hash.argtypes = [c_int, c_int, c_int, ctypes.POINTER(c_dp), c_dp, c_dp]
    lib.hps_leaf_hash.restype = c_int
    lib.hps_leaf_verify.argtypes = [c_int, c_int, c_int, ctypes.POINTER(c_dp), c_dp, c_dp, c_dp]
    lib.hps_leaf_verify.restype = c_int
    lib.hps_leaf_fields.argtypes = [c_int, c_int, c_dp, c_int, c_int, c_dp, c_dp, c_dp, c_dp, c_dp, c_dp, c_dp,
                                    c_dp, c_dp]
    lib.hps_leaf_fields.restype = c_int
    lib.hps_eval_points.argtypes = [c_int, c_int, c_dp, c_int, c_dp, c_dp, c_dp, c_dp, c_dp]
    lib.hps_eval_points.restype = c_int
    lib.hps_gauge_sides.argtypes = [c_int, c_int, c_dp, c_int, c_dp, c_dp, c_dp, c_dp]
    lib.hps_gauge_sides.restype = c_int
    lib.hps_gauge_gather.argtypes = [c_int, c_int, c_dp, c_dp, c_dp, c_int, c_dp, c_int, c_dp]
    lib.hps_gauge_gather.restype = c_int
    _lib = lib
    return lib


class Context:
    """An hps_ctx_t (include/hps_b200.h): the library's side streams, split-K scratch and options
    for one device. Two builds in flight at once use two contexts."""

    def __init__(self, device_index, **options):
        lib = load()
        h = c_dp()
        check(lib.hps_ctx_create(int(device_index), ctypes.byref(h)), "hps_ctx_create")
        self.handle = h
        self.device_index = int(device_index)
        for k, v in options.items():
            self.set(k, v)

    def set(self, name, value):
        opt = globals()["HPS_OPT_" + name.upper()]
        check(load().hps_ctx_set_option(self.handle, opt, int(value)), "hps_ctx_set_option")

    def get(self, name):
        return int(load().hps_ctx_get_option(self.handle, globals()["HPS_OPT_" + name.upper()]))

    def close(self):
        if self.handle is not None and self.handle.value:
            load().hps_ctx_destroy(self.handle)
        self.handle = None

    _as_parameter_ = property(lambda self: self.handle)


_contexts = {}


def context(slot=0, device=None):
    """The shared context `slot` of a device (default: the current CUDA device). Slot k is what a
    k-th concurrent build stream uses (solver.Pipeline); created on first use, kept for the
    process lifetime."""
    import torch

    dev = None if device is None else torch.device(device).index
    dev = torch.cuda.current_device() if dev is None else dev
    key = (dev, slot)
    c = _contexts.get(key)
    if c is None:
        require_device()
        c = _contexts[key] = Context(dev)
    return c


def last_error():
    return load().hps_last_error().decode(errors="replace")


def check(status, what):
    if status != HPS_OK:
        msg = load().hps_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (status {status}): {msg}")


_device_ok = False


def require_device():
    """Fail loudly unless an sm_100 device is usable through the library."""
    global _device_ok
    if _device_ok:
        return
    import torch

    if not torch.cuda.is_available():
        raise NativeError("the HPS B200 path needs a CUDA device (sm_100a); there is no CPU fallback")
    lib = load()
    ma, mi, sms = c_int(), c_int(), c_int()
    check(lib.hps_device_check(ctypes.byref(ma), ctypes.byref(mi), ctypes.byref(sms)), "hps_device_check")
    _device_ok = True


def ptr(t):
    """Device pointer of a C-contiguous tensor (None -> NULL). The kernels assume row-major
    dense storage; a strided view would be silently misread, so it is rejected here."""
    if t is None:
        return ctypes.c_void_p(0)
    if not t.is_contiguous():
        raise NativeError(f"non-contiguous tensor passed to the C ABI: shape {tuple(t.shape)} "
                          f"stride {tuple(t.stride())}")
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
