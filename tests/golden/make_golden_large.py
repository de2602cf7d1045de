"""Golden vectors at the BASELINE sizes, from the REFERENCE itself, with its own self-noise floor.

Test infrastructure. Run in the build container, where /root/reference exists:

    python tests/golden/make_golden_large.py all          # every case below, then `combine`
    python tests/golden/make_golden_large.py run CFG L THREADS   # one reference run (subprocess)
    python tests/golden/make_golden_large.py combine      # fixtures + noise from the runs
    python tests/golden/make_golden_large.py hashes       # L = 8, 9 layout hashes

A `run` pins OMP_NUM_THREADS / OPENBLAS_NUM_THREADS BEFORE numpy is imported (OpenBLAS ignores a
later setting), builds with hpsolve.solver.build(..., switch_threshold=None) (reference
solver.py:250-289) and solves one seeded boundary vector with hpsolve.solver.solve (solver.py:303-316).
It keeps, for the whole problem: root T, and L1 u[I_e] for every leaf (the null-mode-invariant
solution). Each case runs twice: all cores and 2 threads. `combine` writes
tests/golden/large_cfg{c}_L{L}.npz holding
  rows, root_T_rows   16 seeded rows of root T (all-cores run)
  G, root_T_sketch    root T @ G for a seeded 4-column Gaussian G
  leaves, L1u         L1 u[I_e] on a seeded subset of 4096 leaves (heap order of leaves)
  F                   the boundary vector (root.I_e order)
  noise_T, noise_sketch, noise_L1u   max-relative difference of each quantity between the
                      two thread counts, over the WHOLE problem (rows / sketch / all leaves)
  noise_T_sub, noise_L1u_sub         the same over the stored subset
  threads             the two thread counts; runtime_s of each run
The GPU tests gate at max(BASELINE tolerance, 10 x noise) (SURVEY.md §8c self-noise rule).
"""

import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")
WORK = os.environ.get("HPS_GOLDEN_WORK", "/tmp/hps_golden")
CASES = [(1, 4), (2, 6), (3, 7), (5, 8), (4, 8)]
SEED_F = 21
N_ROWS = 16
N_LEAVES = 4096

if __name__ == "__main__" and len(sys.argv) >= 5 and sys.argv[1] == "run":
    os.environ["OMP_NUM_THREADS"] = sys.argv[4]
    os.environ["OPENBLAS_NUM_THREADS"] = sys.argv[4]
    os.environ["MKL_NUM_THREADS"] = sys.argv[4]

import numpy as np  # noqa: E402

sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")


def _paths(cfg, L, thr):
    base = os.path.join(WORK, f"cfg{cfg}_L{L}_t{thr}")
    return base + "_rootT.npy", base + "_L1u.npy", base + "_meta.json"


def run(cfg, L, thr):
    from hpsolve import grid, leafops, solver  # the reference
    from paper_1307_2665_b200 import problems  # generators only (shared with the GPU side)
    os.makedirs(WORK, exist_ok=True)
    co = problems.coefficients(cfg)
    ref = leafops.CoefficientField(**{n: getattr(co, n) for n in ("c11", "c12", "c22", "c1", "c2", "c")})
    t0 = time.perf_counter()
    t, n = grid.build_tree(grid.Rectangle(0, 1, 0, 1), L, 16)
    t1 = time.perf_counter()
    st = solver.build(t, n, ref, switch_threshold=None)
    t2 = time.perf_counter()
    F = np.asarray(problems.boundary_data(cfg, n.points[t.root.I_e], seed=SEED_F, batch=1)).reshape(-1)
    u = solver.solve(st, F)
    t3 = time.perf_counter()
    geom = st.geometry
    Ie = np.stack([b.I_e for b in t.leaves()])
    L1u = np.einsum("rc,lc->lr", geom.L1, u[Ie])
    pT, pU, pM = _paths(cfg, L, thr)
    np.save(pT, st.root_T.dense)
    np.save(pU, L1u)
    with open(pM, "w") as f:
        json.dump({"tree_s": t1 - t0, "build_s": t2 - t1, "solve_s": t3 - t2, "threads": thr,
                   "F": F.tolist()}, f)
    print(f"cfg{cfg} L{L} t{thr}: tree {t1 - t0:.1f}s build {t2 - t1:.1f}s solve {t3 - t2:.2f}s", flush=True)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def combine(cfg, L, hi, lo):
    pT, pU, pM = _paths(cfg, L, hi)
    qT, qU, qM = _paths(cfg, L, lo)
    T = np.load(pT, mmap_mode="r")
    T2 = np.load(qT, mmap_mode="r")
    U, U2 = np.load(pU), np.load(qU)
    mh, ml = json.load(open(pM)), json.load(open(qM))
    n = T.shape[0]
    rng = np.random.default_rng(1000 + cfg)
    rows = np.sort(rng.choice(n, size=min(N_ROWS, n), replace=False))
    G = rng.standard_normal((n, 4))
    leaves = np.sort(rng.choice(U.shape[0], size=min(N_LEAVES, U.shape[0]), replace=False))
    sk, sk2 = T @ G, T2 @ G
    tmax = max(float(np.abs(T[i0:i0 + 1024]).max()) for i0 in range(0, n, 1024))
    tdiff = max(float(np.abs(T[i0:i0 + 1024] - T2[i0:i0 + 1024]).max()) for i0 in range(0, n, 1024))
    out = {
        "rows": rows, "root_T_rows": np.ascontiguousarray(T[rows]), "G": G, "root_T_sketch": sk,
        "leaves": leaves, "L1u": U[leaves], "F": np.array(mh["F"]),
        "noise_T": np.array(tdiff / tmax), "noise_sketch": np.array(_rel(sk2, sk)),
        "noise_L1u": np.array(_rel(U2, U)),
        "noise_T_sub": np.array(_rel(np.asarray(T2[rows]), np.asarray(T[rows]))),
        "noise_L1u_sub": np.array(_rel(U2[leaves], U[leaves])),
        "threads": np.array([hi, lo]), "build_s": np.array([mh["build_s"], ml["build_s"]]),
        "solve_s": np.array([mh["solve_s"], ml["solve_s"]]),
    }
    np.savez_compressed(os.path.join(HERE, f"large_cfg{cfg}_L{L}.npz"), **out)
    print(f"cfg{cfg} L{L}: noise T {out['noise_T']:.2e} sketch {out['noise_sketch']:.2e} "
          f"L1u {out['noise_L1u']:.2e} (subset {out['noise_L1u_sub']:.2e}); build {mh['build_s']:.0f}s "
          f"/ {ml['build_s']:.0f}s", flush=True)


def hashes():
    sys.path.insert(0, HERE)
    import make_golden as mg
    path = os.path.join(HERE, "tree_hashes.json")
    h = json.load(open(path))
    for L in (8, 9):
        t0 = time.perf_counter()
        h[f"L{L}_q16"] = mg.digest(mg.tree_arrays((0, 1, 0, 1), L, 16))
        print(f"L{L} hash in {time.perf_counter() - t0:.0f}s", flush=True)
        with open(path, "w") as f:
            json.dump(h, f, indent=1)


def main():
    cmd = sys.argv[1]
    hi = str(os.cpu_count())
    if cmd == "run":
        run(int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
    elif cmd == "combine":
        for cfg, L in CASES:
            if os.path.exists(_paths(cfg, L, "2")[2]) and os.path.exists(_paths(cfg, L, hi)[2]):
                combine(cfg, L, hi, "2")
    elif cmd == "hashes":
        hashes()
    elif cmd == "all":
        for cfg, L in CASES:
            for thr in (hi, "2"):
                if not os.path.exists(_paths(cfg, L, thr)[2]):
                    subprocess.run([sys.executable, __file__, "run", str(cfg), str(L), thr], check=True)
            combine(cfg, L, hi, "2")
            for thr in (hi, "2"):  # root T files are GBs; keep the disk clean
                os.remove(_paths(cfg, L, thr)[0])
        hashes()


if __name__ == "__main__":
    main()
