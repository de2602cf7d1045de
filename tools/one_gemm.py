import sys
sys.path.insert(0, ".")
import torch
from paper_1307_2665_b200 import _native
lib = _native.load()
M, N, K, B = (int(x) for x in sys.argv[1:5])
A = torch.randn(B, M, K, dtype=torch.float64, device="cuda"); Bm = torch.randn(B, K, N, dtype=torch.float64, device="cuda")
C = torch.empty(B, M, N, dtype=torch.float64, device="cuda")
for _ in range(3):
    _native.check(lib.hps_dgemm_batched(_native.context(), M, N, K, B, 1.0, _native.ptr(A), K, M*K, _native.ptr(Bm), N, K*N, None, 0, 0.0, _native.ptr(C), N, M*N, _native.stream_ptr()), "g")
torch.cuda.synchronize(); print("ok")
