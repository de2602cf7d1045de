set -u
mkdir -p gpurun_out
python - <<'PY' > gpurun_out/nan_debug.txt 2>&1
import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from paper_1307_2665_b200 import _native
lib = _native.load()
M, N, K, B = 256, 1040, 512, 2
rng = np.random.default_rng(14)
A = rng.standard_normal((B, M, K)); Bm = rng.standard_normal((B, K, N))
A[1, 5, 7] = np.inf; A[0, 9, :] = 0.0
for mb in (1, 8192):
    cx = _native.Context(0, emu_min_work=1, emu_min_k=16, emu_slices=0, emu_moduli=14, emu_scratch_mb=mb)
    tA = torch.tensor(A, device="cuda"); tB = torch.tensor(Bm, device="cuda")
    tC = torch.zeros((B, M, N), dtype=torch.float64, device="cuda")
    _native.check(lib.hps_dgemm_batched(cx, M, N, K, B, -2.0, _native.ptr(tA), K, M * K, _native.ptr(tB), N, K * N, None, 0, 0.0, _native.ptr(tC), N, M * N, _native.stream_ptr()), "g")
    C = tC.cpu().numpy(); cx.close()
    bad = np.argwhere(np.isnan(C))
    print(mb, "nan count", len(bad), "rows", sorted(set(map(tuple, bad[:, :2].tolist())))[:10], "cols", sorted(set(bad[:, 2].tolist()))[:20])
    ref = -2.0 * np.einsum("bmk,bkn->bmn", A, Bm)
    ok = ~np.isnan(C); ok[1, 5] = False
    print("  max abs diff where finite:", np.abs(C - ref)[ok].max())
PY
cat gpurun_out/nan_debug.txt
for s in "4096 4096 1024 64" "8192 8192 2048 16" "32768 32768 8192 1"; do
  timeout 300 python tools/emu_profile.py $s 14 0 > gpurun_out/prof_$(echo $s | tr ' ' _).txt 2>&1; cat gpurun_out/prof_$(echo $s | tr ' ' _).txt | head -14
  timeout 300 python tools/emu_profile.py $s 0 8 | head -12
done
