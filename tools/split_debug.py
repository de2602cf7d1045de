"""Dev probe: modular emulation with the FP64-pipe residues (split 0) vs the integer/MMA ones (split 1)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1307_2665_b200 import _native
lib = _native.load()
M, N, K, B, moduli = (int(x) for x in sys.argv[1:6])
rng = np.random.default_rng(M + moduli)
A = rng.standard_normal((B, M, K)) * np.exp2(rng.integers(-20, 20, (B, M, 1)))
Bm = rng.standard_normal((B, K, N)) * np.exp2(rng.integers(-20, 20, (B, 1, N)))
outs = []
for split in (0, 1, 1):
    cx = _native.Context(0, emu_min_work=1, emu_min_k=16, emu_slices=0, emu_moduli=moduli, emu_split=split)
    tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(Bm).cuda()
    tC = torch.zeros((B, M, N), dtype=torch.float64, device="cuda")
    _native.check(lib.hps_dgemm_batched(cx, M, N, K, B, 1.0, _native.ptr(tA), K, M * K, _native.ptr(tB), N, K * N, None, 0, 0.0,
                                        _native.ptr(tC), N, M * N, _native.stream_ptr()), "gemm")
    outs.append(tC.cpu().numpy())
    cx.close()
ref = np.einsum("bmk,bkn->bmn", A.astype(np.longdouble), Bm.astype(np.longdouble))
scale = np.abs(A).max(axis=2)[:, :, None] * np.abs(Bm).max(axis=1)[:, None, :] * K
for i, o in enumerate(outs):
    print("split", (0, 1, 1)[i], "err", float((np.abs(o - ref) / scale).max()))
d = outs[0] != outs[1]
print("differ 0 vs 1:", d.sum(), "of", d.size, "; 1 vs 1:", (outs[1] != outs[2]).sum())
if d.any():
    bb, rr, cc = np.nonzero(d)
    print("batches", np.unique(bb), "rows", np.unique(rr)[:20], len(np.unique(rr)), "cols", np.unique(cc)[:20], len(np.unique(cc)))
    i = 0
    print(outs[0][bb[i], rr[i], cc[i]], outs[1][bb[i], rr[i], cc[i]], float(ref[bb[i], rr[i], cc[i]]))
