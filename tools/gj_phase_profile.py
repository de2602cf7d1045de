"""Owner-warp phase cycles of k_gj_blk (tools/libhps_b200_prof.so built with -DHPS_GJ_PROFILE)."""
import os, sys, ctypes
os.environ["HPS_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhps_b200_prof.so")
sys.path.insert(0, ".")
import torch
from paper_1307_2665_b200 import _native
lib = _native.load()
for n in (32, 64, 128):
    A = torch.randn(1, n, n, dtype=torch.float64, device="cuda") + n * torch.eye(n, dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.hps_inverse_workspace_bytes(n, 1), dtype=torch.uint8, device="cuda")
    st = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    buf = (ctypes.c_longlong * 8)()
    X = A.clone()
    lib.hps_inverse_batched(_native.context(), n, 1, _native.ptr(X), n, n * n, _native.ptr(ws), ws.numel(), _native.ptr(st), _native.stream_ptr())
    torch.cuda.synchronize()
    lib.hps_debug_gj_profile(buf, 1)
    X = A.clone()
    lib.hps_inverse_batched(_native.context(), n, 1, _native.ptr(X), n, n * n, _native.ptr(ws), ws.numel(), _native.ptr(st), _native.stream_ptr())
    torch.cuda.synchronize()
    lib.hps_debug_gj_profile(buf, 0)
    nb = n // 8 - 1
    names = ["stage A_P", "update own tile", "panel (8 pivots)", "update other tile", "barrier wait", "block total"]
    print(f"n={n}: cycles per block (owner warp lane 0):", ", ".join(f"{nm} {buf[i] / nb:.0f}" for i, nm in enumerate(names)),
          f"| first panel alone {buf[6]}")
