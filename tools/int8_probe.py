"""int8 x int8 -> int32 GEMM throughput on this GPU through cuBLASLt (torch._int_mm): feasibility
probe for an FP64-by-int8-slices (Ozaki) emulation of the big merge GEMMs (dev tool)."""
import sys
import torch

torch.manual_seed(0)
for (M, N, K) in [(8192, 8192, 8192), (16384, 16384, 8192), (32768, 32768, 8192), (32768, 8192, 8192 * 4)]:
    a = torch.randint(-64, 64, (M, K), dtype=torch.int8, device="cuda")
    bt = torch.randint(-64, 64, (N, K), dtype=torch.int8, device="cuda")
    b = bt.t()  # column-major K x N
    for _ in range(2):
        c = torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 5
    for _ in range(n):
        c = torch._int_mm(a, b)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{M}x{N}x{K}: {ms:.2f} ms, {2.0 * M * N * K / ms / 1e9:.0f} TOPS", flush=True)
    if M == 8192:
        ref = (a[:256].double() @ b[:, :256].double())
        print("exact:", bool((c[:256, :256].double() == ref).all()))
    del a, b, bt, c
    torch.cuda.empty_cache()
