"""Our DMMA GEMM vs cuBLAS (torch.bmm) on the merge shapes of cfg2 (L=6) and cfg5 top depths (dev tool)."""
import sys
sys.path.insert(0, ".")
import torch
from tools.bench_inverse import t_gemm
shapes = []
for (n3, ne, b) in [(1024, 4096, 1), (512, 3072, 2), (512, 2048, 4), (256, 1536, 8), (256, 1024, 16), (128, 768, 32),
                    (4096, 16384, 4), (2048, 12288, 8)]:
    shapes.append((ne, ne, n3, b))   # T = blk + C S
    shapes.append((n3, ne, n3, b))   # S = X^-1 R
for M, N, K, b in shapes:
    t_gemm(M, N, K, b)
