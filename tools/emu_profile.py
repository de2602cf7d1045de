"""Per-kernel device times of one emulated (or DMMA) merge-shaped GEMM through hps_dgemm_batched,
from torch.profiler (CUPTI): which of scales / residues / int8 products / reconstruction dominate
(dev tool). Usage: python tools/emu_profile.py M N K batch [moduli slices scratch_mb engine tile_group split]"""
import sys
from collections import defaultdict

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1307_2665_b200 import _native

lib = _native.load()
M, N, K, B = (int(x) for x in sys.argv[1:5])
moduli = int(sys.argv[5]) if len(sys.argv) > 5 else 14
slices = int(sys.argv[6]) if len(sys.argv) > 6 else 0
scratch = int(sys.argv[7]) if len(sys.argv) > 7 else 8192
engine = int(sys.argv[8]) if len(sys.argv) > 8 else 0
group = int(sys.argv[9]) if len(sys.argv) > 9 else 0
split = int(sys.argv[10]) if len(sys.argv) > 10 else 1
cx = _native.Context(0, emu_moduli=moduli, emu_slices=slices, emu_scratch_mb=scratch, emu_engine=engine,
                     emu_tile_group=group, emu_min_k=16, emu_split=split)
A = torch.randn(B, M, K, dtype=torch.float64, device="cuda")
Bm = torch.randn(B, K, N, dtype=torch.float64, device="cuda")
C = torch.empty(B, M, N, dtype=torch.float64, device="cuda")


def run():
    _native.check(lib.hps_dgemm_batched(cx, M, N, K, B, 1.0, _native.ptr(A), K, M * K, _native.ptr(Bm), N, K * N, None, 0,
                                        0.0, _native.ptr(C), N, M * N, _native.stream_ptr()), "gemm")


for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    run()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 3
fl = 2.0 * M * N * K * B
print(f"M={M} N={N} K={K} B={B} moduli={moduli} slices={slices} engine={engine} group={group}: {ms:.3f} ms, {fl / ms / 1e9:.1f} TF/s FP64-equivalent")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        agg[ev.name][0] += 1
        agg[ev.name][1] += ev.device_time_total / 1e3
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {t:9.3f} ms  x{n:<4d} {name[:110]}")
if M * N * B <= 1 << 26:
    ref = (A.cpu().numpy() @ Bm.cpu().numpy())
    print("max rel err vs numpy:", float(np.abs(C.cpu().numpy() - ref).max() / np.abs(ref).max()))
cx.close()
