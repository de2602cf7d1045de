"""cuBLAS DGEMM (torch.matmul fp64) throughput on the box: the FP64 roofline denominator."""
import json, time, torch
res = {}
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = 2 * n**3 / (best * 1e-3) / 1e12
    print(f"dgemm n={n}: {best:.3f} ms {res[n]:.2f} TFLOP/s", flush=True)
# sustained 4 s
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
torch.cuda.synchronize(); t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4:
    c = a @ b; cnt += 1
    if cnt % 8 == 0: torch.cuda.synchronize()
e1.record(); e1.synchronize()
sus = 2 * n**3 * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(f"dgemm sustained n=8192: {sus:.2f} TFLOP/s")
print(json.dumps({"fp64_tflops_burst": max(res.values()), "fp64_tflops_sustained": sus}))
