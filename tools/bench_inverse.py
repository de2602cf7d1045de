"""Micro-benchmark of the batched interface inverse and of the DMMA GEMM (dev tool)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1307_2665_b200 import _native
lib = _native.load()
def t_inv(n, batch, reps=5):
    A = torch.randn(batch, n, n, dtype=torch.float64, device="cuda") + n * torch.eye(n, dtype=torch.float64, device="cuda")
    X = A.clone()
    ws = torch.empty(lib.hps_inverse_workspace_bytes(n, batch), dtype=torch.uint8, device="cuda")
    st = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    def run():
        X.copy_(A)
        _native.check(lib.hps_inverse_batched(_native.context(), n, batch, _native.ptr(X), n, n * n, _native.ptr(ws), ws.numel(), _native.ptr(st), _native.stream_ptr()), "inv")
    run(); torch.cuda.synchronize()
    err = float((torch.bmm(A, X) - torch.eye(n, dtype=torch.float64, device="cuda")).abs().max())
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        X.copy_(A); e0.record()
        _native.check(lib.hps_inverse_batched(_native.context(), n, batch, _native.ptr(X), n, n * n, _native.ptr(ws), ws.numel(), _native.ptr(st), _native.stream_ptr()), "inv")
        e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"inverse n={n:5d} batch={batch:6d}: {best*1e3:9.1f} us  {2*n**3*batch/best/1e9:8.2f} TF/s  |AX-I|={err:.1e}", flush=True)
def t_gemm(M, N, K, batch, reps=5):
    A = torch.randn(batch, M, K, dtype=torch.float64, device="cuda"); B = torch.randn(batch, K, N, dtype=torch.float64, device="cuda")
    C = torch.empty(batch, M, N, dtype=torch.float64, device="cuda")
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps + 1):
        e0.record()
        _native.check(lib.hps_dgemm_batched(_native.context(), M, N, K, batch, 1.0, _native.ptr(A), K, M*K, _native.ptr(B), N, K*N, None, 0, 0.0, _native.ptr(C), N, M*N, _native.stream_ptr()), "g")
        e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    tc = 1e9
    for _ in range(reps + 1):
        e0.record(); torch.bmm(A, B, out=C); e1.record(); e1.synchronize(); tc = min(tc, e0.elapsed_time(e1))
    fl = 2 * M * N * K * batch
    print(f"gemm {M}x{N}x{K} b={batch}: ours {best*1e3:8.1f} us {fl/best/1e9:6.2f} TF/s | cublas {tc*1e3:8.1f} us {fl/tc/1e9:6.2f} TF/s", flush=True)
if __name__ == "__main__":
    for n, b in [(16, 1), (16, 2048), (32, 1), (32, 1024), (64, 1), (64, 256), (128, 1), (128, 64), (128, 148), (256, 1), (512, 1), (1024, 1), (2048, 1)]:
        t_inv(n, b)
    if "inv" in sys.argv:
        sys.exit(0)
    for (M, N, K, b) in [(4096, 4096, 1024, 1), (3072, 3072, 512, 2), (2048, 2048, 512, 4), (1024, 1024, 256, 16), (512, 512, 128, 64), (256, 256, 64, 256), (128, 128, 32, 1024), (96, 96, 16, 2048),
                          (1024, 4096, 1024, 1), (512, 2048, 512, 4), (8192, 8192, 8192, 1), (512, 512, 512, 1), (256, 256, 256, 1)]:
        t_gemm(M, N, K, b)
