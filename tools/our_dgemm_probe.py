"""One DGEMM through hps_dgemm_batched (4096x4096x1024) for ncu inspection (dev tool)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_1307_2665_b200 import _native
lib = _native.load()
A = torch.randn(4096, 1024, dtype=torch.float64, device="cuda")
B = torch.randn(1024, 4096, dtype=torch.float64, device="cuda")
C = torch.empty(4096, 4096, dtype=torch.float64, device="cuda")
for _ in range(3):
    _native.check(lib.hps_dgemm_batched(_native.context(), 4096, 4096, 1024, 1, 1.0, _native.ptr(A), 1024, 0, _native.ptr(B), 4096, 0, None, 0,
                                        0.0, _native.ptr(C), 4096, 0, _native.stream_ptr()), "g")
torch.cuda.synchronize()
