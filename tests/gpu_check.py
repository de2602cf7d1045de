"""Quick GPU validation of the CUDA path against the oracle (dev tool; the formal gates are tests/)."""
import sys, time
import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from oracle import hps_oracle as O
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import _native, problems, solver


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def check_gemm():
    lib = _native.load()
    rng = np.random.default_rng(0)
    for (M, N, K, B) in [(64, 64, 16, 1), (96, 96, 16, 3), (256, 512, 128, 2), (1000, 130, 64, 1), (128, 128, 32, 200)]:
        A = rng.standard_normal((B, M, K)); Bm = rng.standard_normal((B, K, N)); C = rng.standard_normal((B, M, N))
        tA, tB, tC = (torch.from_numpy(x).cuda() for x in (A, Bm, C))
        st = lib.hps_dgemm_batched(_native.context(), M, N, K, B, 0.5, _native.ptr(tA), K, M * K, _native.ptr(tB), N, K * N, None, 0, 2.0,
                                   _native.ptr(tC), N, M * N, _native.stream_ptr())
        _native.check(st, "gemm")
        ref = 0.5 * A @ Bm + 2.0 * C
        print(f"gemm M={M} N={N} K={K} B={B}: rel {rel(tC.cpu().numpy(), ref):.2e}")
    # gather
    M, N, K = 48, 64, 32
    U = rng.standard_normal((500, N)); idx = rng.integers(0, 500, K).astype(np.int32); A = rng.standard_normal((M, K))
    C = np.zeros((M, N))
    tA, tU, tC, ti = torch.from_numpy(A).cuda(), torch.from_numpy(U).cuda(), torch.from_numpy(C).cuda(), torch.from_numpy(idx).cuda()
    _native.check(lib.hps_dgemm_batched(_native.context(), M, N, K, 1, 1.0, _native.ptr(tA), K, 0, _native.ptr(tU), N, 0, _native.ptr(ti), 0, 0.0,
                                        _native.ptr(tC), N, 0, _native.stream_ptr()), "gemm gather")
    print(f"gemm gather rel {rel(tC.cpu().numpy(), A @ U[idx]):.2e}")


def coeff_dict(cf):
    return {n: getattr(cf, n) for n in O.COEFF_NAMES}


def check_cfg(cfg, L, b=3):
    c = problems.CONFIGS[cfg]
    cf = c.coefficients()
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
    t0 = time.time()
    st = solver.build(tree, nodes, cf, switch_threshold=None, keep_level_T=True)
    torch.cuda.synchronize()
    tg = time.time() - t0
    otree = O.build_tree((0, 1, 0, 1), L, 16)
    t0 = time.time()
    ost = O.build(otree, coeff_dict(cf), keep_T=True)
    to = time.time() - t0
    out = [f"cfg{cfg} L={L}: gpu {tg:.2f}s oracle {to:.2f}s groups {st.n_leaf_groups}"]
    out.append(f"leafT {rel(st.T_leaf_groups.cpu().numpy(), ost.T_groups):.1e}")
    out.append(f"psi {rel(st.psi_groups.cpu().numpy(), ost.psi_groups):.1e}")
    out.append(f"cond {rel(st._cond.cpu().numpy(), ost.cond):.1e}")
    worst = 0.0
    for d in range(2 * L):
        Td = st.level_T[d].cpu().numpy()
        for k in range(Td.shape[0]):
            worst = max(worst, rel(Td[k], ost.T[(1 << d) - 1 + k]))
    out.append(f"all merged T {worst:.1e}")
    out.append(f"rootT {rel(st.root_T.dense, ost.root_T):.1e}")
    pts = nodes.points[tree.root.I_e]
    F = problems.boundary_data(cfg, pts, seed=1, batch=b)
    u = solver.solve(st, F)
    uo = O.solve(ost, F)
    wg = O.leaf_cheb_boundary(ost, u)
    wo = O.leaf_cheb_boundary(ost, uo)
    out.append(f"L1u {rel(wg, wo):.1e}")
    ex = problems.exact_solution(cfg, nodes.points[:, 0], nodes.points[:, 1], seed=1, batch=b)
    if ex is not None:
        we = O.leaf_cheb_boundary(ost, ex)
        out.append(f"L1u-vs-exact gpu {rel(wg, we):.1e} oracle {rel(wo, we):.1e}")
    print("  ".join(out), flush=True)


if __name__ == "__main__":
    check_gemm()
    for cfg in (1, 2, 3, 4, 5):
        check_cfg(cfg, 2)
    for cfg in (1, 2, 3, 4, 5):
        check_cfg(cfg, 4)
    # timing cfg2 L=6
    c = problems.CONFIGS[2]
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 6, 16)
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.time()
        st = solver.build(tree, nodes, c.coefficients(), switch_threshold=None)
        torch.cuda.synchronize(); t1 = time.time()
        F = torch.from_numpy(problems.boundary_data(2, nodes.points[tree.root.I_e], seed=0)).cuda()
        torch.cuda.synchronize(); t2 = time.time()
        U = solver.solve_device(st, F)
        torch.cuda.synchronize(); t3 = time.time()
        print(f"cfg2 L=6 build {t1-t0:.3f}s solve(b=64) {t3-t2:.4f}s")
