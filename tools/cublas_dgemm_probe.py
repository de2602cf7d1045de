"""One cuBLAS DGEMM (torch.bmm, 4096x4096x1024) for ncu inspection of its kernel (dev tool)."""
import torch
A = torch.randn(1, 4096, 1024, dtype=torch.float64, device="cuda")
B = torch.randn(1, 1024, 4096, dtype=torch.float64, device="cuda")
C = torch.empty(1, 4096, 4096, dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.bmm(A, B, out=C)
torch.cuda.synchronize()
