"""Timing model of the reference's dense CPU path, built from the oracle port (test and
measurement infrastructure: only bench.py's cpu_baseline / --impl reference legs use it; it is
never part of the product path).

The reference (hpsolve, pure numpy/scipy) runs `solver.build(..., switch_threshold=None)`
(reference solver.py:250-289: leaf stage solver.py:196-246, one `split_indices` + `merge_dtn` per
box, merge.py:68-119) and then b single-RHS `solver.solve` sweeps (solver.py:303-316). Where a whole
step fits in a bounded time, `full_run` times exactly that, through the oracle port
(oracle/hps_oracle.py, which restates those calls with the same LAPACK routines). Where it does not
(config 5: 6.8e13 flop of merges plus 256 sweeps over 34 GB of S), `model` measures a bounded
sample and extrapolates:

* leaf stage: `leaf_operators` on k of the n_g distinct groups (median of 3), times n_g / k;
* merges: every depth whose single merge is at most `cap` flop is MEASURED: one real merge chain
  (each depth merges two copies of the previous depth's T, so shapes and index maps are exactly
  the tree's), each timed as m consecutive `split_indices` + `merge_dtn` calls (m large enough
  for a stable timer), median of 3, times 2^d. Above the cap, a merge is SCALED from the depth two
  below (same aspect ratio n3 : ne, 8x the flops) by the flop ratio, since BLAS-3 at n3 >= 1024
  runs at its saturated rate;
* solve: per depth, `u[I_i] = S u[I_e]` on the tree's real index lists, cycling through enough
  distinct S matrices that they stream from DRAM as the reference's 2^d distinct S do, times
  2^d; times b right-hand sides (the reference solve is single-RHS, solver.py:298-299).

`validate` compares the model with `full_run` at configurations that fit (bench.py
--validate-reference-model); profiles/reference_model_validation_*.json holds the result.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import hps_oracle as O

CAP_FLOP = 2e11  # largest single merge timed directly
MIN_FLOP_PER_TIMING = 5e8  # small merges are timed in runs of at least this much work
SOLVE_POOL_BYTES = 192 << 20  # distinct S per depth, to stream them like the reference's


def _median3(fn):
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def merge_flop(n3, ne):
    return 2.0 / 3.0 * n3 ** 3 + 2.0 * n3 ** 2 * ne + 2.0 * n3 * ne ** 2


def _setup(cfg, L, q):
    from paper_1307_2665_b200 import problems  # generators only (shared seeded inputs)
    co = problems.coefficients(cfg)
    coeffs = {n: getattr(co, n) for n in O.COEFF_NAMES}
    tree = O.build_tree((0.0, 1.0, 0.0, 1.0), L, q)
    geom = O.Geometry(q, tree.leaf_width, tree.leaf_height)
    fields = O.sample_coefficients(coeffs, tree, geom)
    reps, gid = O.group_leaves(fields, len(tree.leaves))
    return tree, geom, fields, reps, gid


def _boundary(cfg, tree, b, seed=0):
    from paper_1307_2665_b200 import problems
    F = np.asarray(problems.boundary_data(cfg, tree.points[tree.I_e[0]], seed=seed, batch=b))
    return F.reshape(F.shape[0], -1)


class Model:
    """One bounded sample of the reference step; `measure()` returns seconds and a breakdown."""

    def __init__(self, cfg, L, b, q=16, cap=CAP_FLOP, max_groups=128):
        self.cfg, self.L, self.b, self.q, self.cap = cfg, L, b, q, cap
        self.tree, self.geom, self.fields, self.reps, self.gid = _setup(cfg, L, q)
        self.k = min(len(self.reps), max_groups)
        self.maps = {}
        for d in range(2 * L):
            box = (1 << d) - 1
            a, c = self.tree.child_a[box], self.tree.child_b[box]
            self.maps[d] = (self.tree.I_e[a], self.tree.I_e[c], self.tree.I_i[box])

    def measure(self):
        tree, L, q = self.tree, self.L, self.q
        ng = len(self.reps)
        t_leaf1 = _median3(lambda: O.leaf_operators(self.geom, self.fields, self.reps[:self.k]))
        _, Tg, _ = O.leaf_operators(self.geom, self.fields, self.reps[:1])
        t_leaf = t_leaf1 * ng / self.k
        per_merge, how, S_of = {}, {}, {}
        T_child = Tg[0]
        for d in range(2 * L - 1, -1, -1):
            n3, ne = O.depth_sizes(L, q, d)
            f = merge_flop(n3, ne)
            if f <= self.cap and T_child is not None:
                Ie_a, Ie_b, I_i = self.maps[d]
                m = int(min(1 << d, max(1, np.ceil(MIN_FLOP_PER_TIMING / f))))
                Tc = T_child

                def run(m=m, Tc=Tc, Ie_a=Ie_a, Ie_b=Ie_b, I_i=I_i):
                    for _ in range(m):
                        j1a, j2b, j3a, j3b = O.split_indices(Ie_a, Ie_b, I_i)  # per box, as merge.py:68
                        out = O.merge_dtn(Tc, Tc, j1a, j2b, j3a, j3b)
                    return out
                per_merge[d] = _median3(run) / m
                how[d] = "measured"
                S, T_child = run(1)
                S_of[d] = S
            else:
                T_child = None
                n3b, neb = O.depth_sizes(L, q, d + 2)
                per_merge[d] = per_merge[d + 2] * f / merge_flop(n3b, neb)
                how[d] = "scaled from depth %d" % (d + 2)
        t_merge = sum(per_merge[d] * (1 << d) for d in per_merge)
        t_sweep = self._sweep(S_of)
        total = t_leaf + t_merge + self.b * t_sweep
        return total, {
            "t_leaf_s": t_leaf, "t_merge_s": t_merge, "t_solve_s": self.b * t_sweep, "t_sweep_1rhs_s": t_sweep,
            "per_depth_merge_s": {str(d): per_merge[d] * (1 << d) for d in sorted(per_merge)},
            "per_depth_how": {str(d): how[d] for d in sorted(how)},
            "leaf_groups_timed": f"{self.k}/{ng}"}

    def _sweep(self, S_of):
        tree, L, q = self.tree, self.L, self.q
        u = np.zeros(tree.points.shape[0])
        u[tree.I_e[0]] = 1.0
        rng = np.random.default_rng(5)
        t = 0.0
        for d in range(2 * L):
            n3, ne = O.depth_sizes(L, q, d)
            nb = 1 << d
            pool = int(min(nb, max(1, SOLVE_POOL_BYTES // (8 * n3 * ne))))
            base = S_of.get(d)
            Ss = [rng.standard_normal((n3, ne)) * 1e-3 if base is None or i else base for i in range(pool)]
            boxes = [(1 << d) - 1 + (i * max(1, nb // pool)) % nb for i in range(pool)]
            idx = [(tree.I_i[bx], tree.I_e[bx]) for bx in boxes]

            def run():
                for S, (ii, ie) in zip(Ss, idx):
                    u[ii] = S @ u[ie]  # solver.py:315 / SolutionOperator.apply (solver.py:93-97)
            run()  # page the pool in
            t += _median3(run) / pool * nb
            del Ss
        return t


def full_run(cfg, L, b, q=16):
    """The whole reference step through the oracle port: leaf stage + every merge (O.build's
    loop, solver.py:250-289) and b single-RHS sweeps (solver.py:303-316). Coefficient sampling
    and grouping are outside the timed build, as on the GPU side."""
    tree, geom, fields, reps, gid = _setup(cfg, L, q)
    t0 = time.perf_counter()
    Psi, Tg, cond = O.leaf_operators(geom, fields, reps)
    t1 = time.perf_counter()
    store = {bx: Tg[gid[k]] for k, bx in enumerate(tree.leaves)}
    st = O.OracleState()
    st.tree, st.S = tree, {}
    for bx in range(tree.n_boxes - 1, -1, -1):
        a, c = tree.child_a[bx], tree.child_b[bx]
        if a < 0:
            continue
        j1a, j2b, j3a, j3b = O.split_indices(tree.I_e[a], tree.I_e[c], tree.I_i[bx])
        S, T = O.merge_dtn(store.pop(a), store.pop(c), j1a, j2b, j3a, j3b)
        st.S[bx] = S
        store[bx] = T
    t2 = time.perf_counter()
    F = _boundary(cfg, tree, b)
    for j in range(F.shape[1]):
        O.solve(st, F[:, j])
    t3 = time.perf_counter()
    return t3 - t0, {"t_leaf_s": t1 - t0, "t_merge_s": t2 - t1, "t_solve_s": t3 - t2}


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    import numpy
    try:
        import scipy
        sv = scipy.__version__
    except ImportError:
        sv = None
    blas = None
    try:
        cfg = numpy.show_config(mode="dicts")
        blas = cfg.get("Build Dependencies", {}).get("blas", {}).get("name")
    except Exception:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(),
            "omp_threads": os.environ.get("OMP_NUM_THREADS"), "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
            "numpy": numpy.__version__, "scipy": sv, "blas": blas}


def validate(cases=((2, 6, 64), (3, 7, 1)), caps=(CAP_FLOP, 1e9)):
    """Model vs full run, per case; ratio = model / full (want within +-15%)."""
    out = []
    for cfg, L, b in cases:
        t_full, brk_full = full_run(cfg, L, b)
        row = {"cfg": cfg, "L": L, "b": b, "full_s": t_full, "full": brk_full, "model": {}}
        for cap in caps:
            t_mod, brk = Model(cfg, L, b, cap=cap).measure()
            row["model"][f"cap_{cap:.0e}"] = {"s": t_mod, "ratio": t_mod / t_full, "breakdown": brk}
        out.append(row)
    return out
