"""Benchmark: HPS build + batched solve throughput (unknowns/s, fp64) on B200.

Contract (driver-facing): `python bench.py --gpus N --steps K --warmup W [--impl reference]` prints
ONE JSON line on rank 0. A "step" is one pass of the hot path: leaf stage -> every merge level ->
one batched downward solve of b boundary vectors. The default workload is the largest BASELINE
configuration that fits one B200: config 5 (convection-diffusion beta = 1000, 512 x 512 leaves,
p = 16, 6.7e7 unknowns, b = 256; the north_star target problem). Other configs via --config.

`value`    unknowns / (t_build + t_solve), inputs resident in HBM (coefficient samples of the
           leaf groups, boundary batch), CUDA events per step, L2 flushed (256 MB write)
           between steps outside the timed events.
`e2e`      the same metric through the public API from pinned host memory: prepare() (sampling,
           grouping, H2D) + build_device + check_build + H2D(F) + solve_device + D2H(u).
`roofline` the dominant stage, measured live (CUDA events): achieved FP64 TFLOP/s vs the
           measured cuBLAS DGEMM peak (profiles/fp64_peak_r01.json; MEASURED_PEAKS.json has no
           fp64 entry).
`cpu_baseline` / --impl reference: the reference's dense CPU path (the oracle port, numpy/scipy
           LAPACK, all host cores; oracle/cpu_model.py). Configs 1-2 time whole steps
           (`full_run`); larger ones a bounded sample extrapolated per depth (`Model`, labelled
           "extrapolated": true; validated against whole runs by --validate-reference-model,
           profiles/reference_model_validation_*.json).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

# BLAS threads must be pinned before numpy is imported (OpenBLAS reads them once, at load time)
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
    os.environ.setdefault(_v, str(os.cpu_count()))

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
sys.path.insert(0, HERE)

FP64_PEAK_FILE = os.path.join(HERE, "profiles", "fp64_peak_r01.json")
FP64_PEAK_FALLBACK = 35.47  # TFLOP/s, cuBLAS DGEMM 8192^3 measured on this pool (round 1)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--levels", type=int, default=None, help="override L (exploration only)")
    ap.add_argument("--batch", type=int, default=None, help="override solve batch b")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="enqueue the build eagerly instead of replaying CUDA graphs")
    ap.add_argument("--emu-slices", type=int, default=None,
                    help="FP64 GEMM emulation on the int8 tensor cores, slice scheme: slices per operand (used when "
                         "--emu-moduli is 0)")
    ap.add_argument("--emu-moduli", type=int, default=None,
                    help="FP64 GEMM emulation, modular scheme: moduli (default 14; 0 = slice scheme or, with "
                         "--emu-slices 0, DMMA only)")
    ap.add_argument("--emu-engine", type=int, default=None,
                    help="int8 products of the modular scheme: 0 = the library's tcgen05 kernel (default), 2 = its "
                         "CTA-pair variant, 1 = cuBLASLt")
    ap.add_argument("--emu-min-k", type=int, default=None, help="emulate merge GEMMs with K >= this (default 512)")
    ap.add_argument("--emu-solve", type=int, default=None, help="batched solve through the emulation too (default 0)")
    ap.add_argument("--emu-split", type=int, default=None,
                    help="operand residues on the integer pipes + int8 MMA (1, default) or the FP64 pipe (0)")
    ap.add_argument("--validate-reference-model", action="store_true",
                    help="time whole oracle-port steps at configs 2 (L=6) and 3 (L=7) against the sampled model")
    ap.add_argument("--full-reference", action="store_true",
                    help="reference arm: time whole steps even above the default size limit")
    ap.add_argument("--force-distributed", action="store_true",
                    help="run the subtree/NCCL path even at world size 1 (plumbing check)")
    return ap.parse_args()


def fp64_peak():
    try:
        with open(FP64_PEAK_FILE) as f:
            d = json.load(f)
        return float(d["fp64_tflops_burst"]), "measured cuBLAS DGEMM 8192^3 (profiles/fp64_peak_r01.json)"
    except Exception:
        return FP64_PEAK_FALLBACK, "measured cuBLAS DGEMM 8192^3, round 1 (constant in bench.py)"


def traffic_from_profiles(workload, stage):
    """DRAM read+write bytes per launch of a stage's dominant kernel, from the committed ncu
    captures (profiles/*_ncu_*.json carrying "workload", "stage", "dram_bytes_per_launch"; the
    latest file name wins). Returns (bytes or None, source)."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(HERE, "profiles", "*_ncu_*.json"))):
        try:
            pj = json.load(open(path))
        except Exception:
            continue
        if pj.get("workload") == workload and pj.get("stage") == stage and "dram_bytes_per_launch" in pj:
            best = (path, pj)
    if best is None:
        return None, None
    path, pj = best
    src = (f"profiles/{os.path.basename(path)}: dram read+write per launch of {pj.get('kernel')} (ncu --set full; "
           f"{pj.get('gpu_time_ms', float('nan')):.3f} ms); algorithmic {pj.get('algorithmic_bytes_per_launch', 0):.3g} B")
    return float(pj["dram_bytes_per_launch"]), src


def time_i8_kernel(M, N, K, nz, engine, reps=3):
    """Live CUDA-event timing of the dominant kernel of an emulated merge GEMM: one launch of the
    tcgen05 int8 kernel (hps_i8gemm_mod) on the production panel shape (the output column panel
    width emu.cu picks under the 8 GB scratch cap), random residues, on the current stream. Returns
    (ms per launch, panel width, algorithmic bytes per launch)."""
    import ctypes

    import torch

    from paper_1307_2665_b200 import _native

    lib = _native.load()
    cap = _native.context().get("emu_scratch_mb") << 20
    maxc = max(32, cap // (nz * M))  # as emu_gemm_crt (csrc/emu.cu) sizes its output column panels
    if maxc >= N:
        nc = N
    else:
        npan = -(-N // maxc)
        nc = min(maxc // 256 * 256, (-(-N // npan) + 255) // 256 * 256)
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randint(-128, 128, (nz, M, K), dtype=torch.int8, device="cuda", generator=g)
    B = torch.randint(-128, 128, (nz, N, K), dtype=torch.int8, device="cuda", generator=g)
    R = torch.empty((nz, M, nc), dtype=torch.uint8, device="cuda")
    moduli = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193][:nz]
    mods = (ctypes.c_int * len(moduli))(*moduli)
    st = _native.stream_ptr()

    def launch():
        _native.check(lib.hps_i8gemm_mod(_native.context(), _native.ptr(A), _native.ptr(B), _native.ptr(R), M, N, nc, 0,
                                         K, nz, 1, mods, len(moduli), engine, st), "hps_i8gemm_mod")

    launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    algo = float(nz) * (M * K + nc * K + M * nc)
    del A, B, R
    torch.cuda.empty_cache()
    return ms, nc, algo


def int8_peak():
    """Dense int8 tensor rate: twice the measured bf16 GEMM rate (sm_100 runs int8 / fp8 at 2x bf16;
    NVIDIA nominal 4.5 POPS dense vs 2.25 PFLOP/s bf16)."""
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            return 2.0 * float(json.load(f)["bf16_tflops"]), "2 x MEASURED_PEAKS.json bf16_tflops (int8 = 2x bf16 on sm_100)"
    except Exception:
        return 2.0 * 1590.0, "2 x fallback bf16 1.59 PFLOP/s (B200_PROFILING.md)"


def configure_emulation(args):
    """Apply the --emu-* options to every context slot; return the scheme that runs (csrc/emu.cu)."""
    from paper_1307_2665_b200 import _native

    for name in ("emu_slices", "emu_moduli", "emu_engine", "emu_min_k", "emu_solve", "emu_split"):
        v = getattr(args, name)
        if v is not None:
            for slot in range(4):
                _native.context(slot).set(name, v)
    cx = _native.context()
    moduli, slices = cx.get("emu_moduli"), cx.get("emu_slices")
    engine = cx.get("emu_engine")
    if moduli > 0:
        return {"scheme": "modular", "moduli": moduli, "int8_products_per_gemm": moduli, "engine_id": engine,
                "engine": {0: "hps::i8::k_i8gemm_mod (tcgen05.mma.kind::i8, TMA, TMEM; single CTAs)",
                           2: "hps::i8::k_i8gemm_mod_pair (tcgen05.mma.cta_group::2.kind::i8, TMA, TMEM; CTA pairs)"
                           }.get(engine, "cuBLASLt IMMA"),
                "min_k": cx.get("emu_min_k")}
    if slices > 0:
        return {"scheme": "slices", "slices": slices, "int8_products_per_gemm": slices * (slices + 1) // 2,
                "engine": "cuBLASLt IMMA", "min_k": cx.get("emu_min_k")}
    return {"scheme": "off", "int8_products_per_gemm": 0}


def hbm_peak():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()

    def stop(self):
        self._stop.set()
        if self._th:
            self._th.join(timeout=6)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------------------------
# The reference's CPU path (oracle port) timed on this host: whole steps where they fit, else a
# bounded sample extrapolated per depth (oracle/cpu_model.py)
# ----------------------------------------------------------------------------------------------
L2_NOTE = ("GPU arm: 256 MB L2 flush between timed steps, outside the step events; "
           "the same workload on both arms")
FULL_STEP_MAX_L = 6  # configs 1-2 (<= ~45 s per step on 16 cores): whole steps are timed


class CpuReference:
    def __init__(self, cfg, L, b, q=16, full=None):
        from oracle import cpu_model as M
        self.M, self.cfg, self.L, self.b, self.q = M, cfg, L, b, q
        self.full = (L <= FULL_STEP_MAX_L) if full is None else full
        self.model = None if self.full else M.Model(cfg, L, b, q)

    def step(self):
        """Seconds of one reference step (build + b single-RHS solves), and its breakdown."""
        if self.full:
            return self.M.full_run(self.cfg, self.L, self.b, self.q)
        return self.model.measure()

    def describe(self, brk):
        info = self.M.host_info()
        cores = int(info["openblas_threads"] or os.cpu_count())
        if self.full:
            desc = (f"whole steps of the oracle port (numpy/scipy LAPACK, reference solver.py:250-316): leaf stage, "
                    f"every merge, {self.b} single-RHS sweeps; t_leaf={brk['t_leaf_s']:.2f}s "
                    f"t_merge={brk['t_merge_s']:.2f}s t_solve={brk['t_solve_s']:.2f}s")
        else:
            scaled = [d for d, h in brk["per_depth_how"].items() if h != "measured"]
            desc = (f"bounded sample of the oracle port (numpy/scipy LAPACK), extrapolated per depth "
                    f"(oracle/cpu_model.py): leaf stage on {brk['leaf_groups_timed']} groups; merges at every depth "
                    f"measured (median of 3) except depths {','.join(scaled) or 'none'} (scaled by flops from two "
                    f"depths below); 1-RHS sweep per depth over streaming S, x {self.b}; t_leaf={brk['t_leaf_s']:.2f}s "
                    f"t_merge={brk['t_merge_s']:.2f}s t_solve={brk['t_solve_s']:.2f}s")
        return cores, desc, info


# ----------------------------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    from paper_1307_2665_b200 import problems

    cfg = args.config
    c = problems.CONFIGS[cfg]
    L = args.levels if args.levels is not None else c.L
    b = args.batch if args.batch is not None else c.batch
    q = 16
    unknowns = (4 ** L) * q * q
    workload = f"cfg{cfg}_{c.name}_L{L}_p{q}_b{b}"
    metric = "HPS build and solve unknowns/s (fp64)"

    if args.validate_reference_model:
        from oracle import cpu_model as M
        res = {"host": M.host_info(), "cases": M.validate()}
        print(json.dumps(res))
        return

    if args.impl == "reference":
        if rank != 0:
            return
        ref = CpuReference(cfg, L, b, q, full=True if args.full_reference else None)
        times, brk = [], {}
        for it in range(args.warmup + args.steps):
            t, brk = ref.step()
            if it >= args.warmup:
                times.append(t)
        t = float(np.median(times))
        v = unknowns / t
        cores, desc, info = ref.describe(brk)
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": v, "unit": "unknowns/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "l2": L2_NOTE},
            "cpu_baseline": {"value": v, "unit": "unknowns/s", "cores": cores, "kind": "port", "sample": desc,
                             "extrapolated": not ref.full, "host": info,
                             "steps_s": [float(x) for x in times], "breakdown": brk},
            "e2e": {"value": v, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch
    import paper_1307_2665_b200 as P
    from paper_1307_2665_b200 import _native, solver
    from paper_1307_2665_b200 import work as Wk

    if world > 1 or args.force_distributed:
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", "0")
        dist.init_process_group("nccl", rank=rank, world_size=world)
        return bench_distributed(args, cfg, c, L, b, q, unknowns, workload, metric, rank, world)
    dev = torch.device("cuda")
    lib = _native.load()
    emu = configure_emulation(args)
    tree, nodes = P.build_tree(P.Rectangle(0.0, 1.0, 0.0, 1.0), L, q)
    co = c.coefficients()
    F_host = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0, batch=b)
    if F_host.ndim == 1:
        F_host = F_host[:, None]
    F_dev = torch.from_numpy(np.ascontiguousarray(F_host)).to(dev)
    inp = solver.prepare(tree, nodes, co, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    # ---- device-resident timed steps ----
    # Default: the build (one CUDA graph per stage) and the solve replayed from solver.BuildGraph,
    # inputs already in its static buffers; --no-graph: eager enqueue of the same kernels.
    pivoted = solver.check_build(solver.build_device(inp))  # depths whose fast inverse needs the pivoted LU
    torch.cuda.synchronize()
    graph = None if args.no_graph else solver.BuildGraph(inp, nrhs=b, pivoted=pivoted)
    if graph is not None:
        graph.load(inp, F_dev)

    def step(timeline=None):
        if graph is not None:
            st = graph.replay_build(timeline)
        else:
            st = solver.build_device(inp, timeline=timeline, pivoted=pivoted)
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        U = graph.replay_solve() if graph is not None else solver.solve_device(st, F_dev)
        return st, U, e

    st = U = None
    for _ in range(args.warmup):
        st = U = None  # free the previous step's operators first (L=9: ~50 GB of S + u)
        st, U, _ = step()
    torch.cuda.synchronize()
    if solver.check_build(st):
        raise RuntimeError("a residual check failed on the pivoted path")
    torch.cuda.synchronize()
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clocks.start()
    launches0 = lib.hps_launch_count()
    t_build, t_solve, stages = [], [], {}
    for _ in range(args.steps):
        st = U = None
        flush.fill_(1.0)
        tl = []
        e0 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st, U, e1 = step(tl)
        e2.record()
        e2.synchronize()
        t_build.append(e0.elapsed_time(e1) / 1e3)
        t_solve.append(e1.elapsed_time(e2) / 1e3)
        for name, a, z in tl:
            stages.setdefault(name, []).append(a.elapsed_time(z) / 1e3)
    # a replay does not pass through the library's host-side launch counter: count the captured ones
    launches = graph.launches * args.steps if graph is not None else lib.hps_launch_count() - launches0
    torch.cuda.synchronize()
    clk = clocks.stop()
    tb, ts = float(np.mean(t_build)), float(np.mean(t_solve))
    t_step = tb + ts
    value = unknowns / t_step

    # ---- roofline of the dominant stage ----
    peak, peak_src = fp64_peak()
    stage_flops = {"leaf": inp.ngroups * Wk.leaf_flops(q)}
    # a look-ahead depth also runs its parent's interface inverse (solver.lookahead_depths)
    for d, f in Wk.merge_stage_flops(L, q, solver.lookahead_depths(inp.layout)).items():
        stage_flops[f"merge_d{d}"] = f
    stage_ms = {k: float(np.mean(v)) * 1e3 for k, v in stages.items()}
    dom = max(stage_ms, key=stage_ms.get)
    ach = stage_flops[dom] / (stage_ms[dom] / 1e3) / 1e12
    leaf_kernel = "hps::k_leaf16v3" if q == 16 else "hps::k_leaf"
    if dom == "leaf":
        kernels = leaf_kernel
    else:
        dd = int(dom.split("_d")[-1])
        ahead_set = solver.lookahead_depths(inp.layout)
        kernels = ("hps_merge_level_ahead: R/C gathers, S GEMM, T GEMM (hps::dgemm64_kernel)"
                   + ("; its interface inverse ran in depth %d's look-ahead" % (dd + 1) if dd + 1 in ahead_set
                      else "; deflation + interface inverse (k_gj_blk / recursive block inverse)")
                   + ("; forms and inverts depth %d's interface matrix beside its T GEMM" % (dd - 1)
                      if dd in ahead_set else ""))
    build_flops = sum(stage_flops.values())
    solve_flops = Wk.solve_flops(L, q, b)
    S_bytes = Wk.solve_S_bytes(L, q)
    hpeak, hsrc = hbm_peak()
    t_roof = Wk.build_roofline_seconds(L, q, inp.ngroups, peak, hpeak)
    traffic, traffic_src = traffic_from_profiles(workload, dom)
    roofline = {
        "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak, "traffic": traffic,
        "traffic_source": traffic_src,
        "kernel": dom, "kernels": kernels, "peak_source": peak_src,
        "stage_ms": stage_ms, "build_tflops": build_flops / tb / 1e12, "build_frac": build_flops / tb / 1e12 / peak,
        "build_roofline": {"t_roof_ms": t_roof * 1e3, "t_meas_ms": tb * 1e3, "frac": t_roof / tb,
                           "model": "sum over stages of max(flop/FP64 peak, bytes/HBM peak), SURVEY.md 8d"},
        "solve": {"tflops": solve_flops / ts / 1e12, "frac_fp64": solve_flops / ts / 1e12 / peak,
                  "gbs_S_stream": S_bytes / ts / 1e9, "frac_hbm": S_bytes / ts / 1e9 / hpeak, "hbm_peak_source": hsrc},
    }
    if dom.startswith("merge_d") and emu["int8_products_per_gemm"] > 0:
        dd = int(dom.split("_d")[-1])
        ops = Wk.emulated_int8_ops(L, q, dd, emu["int8_products_per_gemm"], min_k=emu["min_k"])
        if ops > 0:
            # the dominant stage's bulk runs on the int8 tensor cores: its roofline is the int8 rate;
            # its FP64-equivalent rate (the algorithmic FP64 flops over the stage time) goes beside it
            i8peak, i8src = int8_peak()
            i8 = ops / (stage_ms[dom] / 1e3) / 1e12
            if emu["scheme"] == "modular":
                how = (f"{emu['moduli']} int8 products (one per modulus) on {emu['engine']}, residues reduced in its "
                       f"epilogue; hps::k_crt_split_rows/cols (residues), k_crt_accum (CRT reconstruction + merge epilogue)")
            else:
                how = (f"{emu['slices']} slices, {emu['int8_products_per_gemm']} int8 products each on cuBLASLt IMMA; "
                       f"hps::k_emu_split_* / k_emu_accum")
            roofline.update({
                "bound": "tensor", "achieved": i8, "peak": i8peak, "unit": "TOPS (int8)", "frac": i8 / i8peak,
                "peak_source": i8src,
                "kernels": f"{dom}: S and T GEMMs as FP64 emulation on the int8 tensor cores ({how}); interface inverse on DMMA",
                "achieved_basis": f"stage level: int8 operations of {dom}'s emulated GEMMs / the stage's time (splits, "
                                  f"reconstruction and the interface inverse included)",
                "fp64_equivalent": {"achieved_tflops": ach, "fp64_dmma_peak_tflops": peak, "ratio_to_fp64_peak": ach / peak,
                                    "note": "algorithmic FP64 flops of the stage / stage time"}})
            if emu["scheme"] == "modular" and emu.get("engine_id", 1) != 1:
                # the dominant kernel itself, timed live: one launch of the int8 kernel on this stage's
                # largest product (the T GEMM: ne x ne x n3, one output column panel, all moduli)
                n3, ne = Wk.depth_sizes(L, q, dd)
                kms, nc, algo = time_i8_kernel(ne, ne, n3, emu["moduli"], emu["engine_id"])
                kt = 2.0 * ne * nc * n3 * emu["moduli"] / (kms / 1e3) / 1e12
                ktraffic, ksrc = traffic_from_profiles(workload, dom + "_i8")
                roofline["kernel_live"] = {
                    "kernel": emu["engine"], "shape": f"{ne} x {nc} (panel of {ne}) x {n3}, {emu['moduli']} moduli",
                    "ms_per_launch": kms, "achieved": kt, "peak": i8peak, "unit": "TOPS (int8)", "frac": kt / i8peak,
                    "frac_of_nominal": kt / 4500.0,
                    "nominal_note": "NVIDIA's dense int8 figure for B200 is 4.5 POPS at boost clock; the measured "
                                    "peak used here (2 x the measured bf16 GEMM rate) reflects the clocks this "
                                    "pool's power cap allows under a sustained tensor load",
                    "algorithmic_bytes_per_launch": algo, "achieved_gbs": algo / (kms / 1e3) / 1e9,
                    "traffic": ktraffic, "traffic_source": ksrc,
                    "basis": "CUDA events around hps_i8gemm_mod launches on the bench stream, after the timed steps"}
                roofline.update({"achieved": kt, "frac": kt / i8peak, "traffic": ktraffic, "traffic_source": ksrc,
                                 "kernel": f"{dom}_i8: {emu['engine']}",
                                 "achieved_basis": "the dominant kernel alone (kernel_live); the stage-level rate is "
                                                   "stage_int8_tops",
                                 "stage_int8_tops": i8})
    # ---- end-to-end through the public API (solver.Pipeline), pinned host memory ----
    # Every step is one full problem: host sampling + grouping of the coefficients, their H2D
    # upload, the build, the H2D of the boundary data, the batched solve and the D2H of u. The
    # pipeline overlaps the host work of step i+1 with the device work of step i, and step i's
    # device work with step i+1's (two compute streams).
    launch_mode = ("CUDA graphs (solver.BuildGraph: one per build stage + one for the solve)"
                   if graph is not None else "eager")
    st = U = graph = None  # the device leg's captured state goes before the pipeline captures its own
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    pin_F = torch.from_numpy(np.ascontiguousarray(F_host)).pin_memory()
    pipe = solver.Pipeline(tree, nodes, device=dev, reuse_graphs=not args.no_graph)
    st = U = None
    # a stream of problems (about 3 s of device time, 5..20 problems): pipeline fill and drain are
    # inside the total; latency_s below is one problem alone
    n_e2e = min(20, max(5, int(3.0 / max(t_step, 1e-6))))
    for U, st in pipe.run([(co, pin_F)] * n_e2e):
        st = None
    st = U = None
    # two timed passes over the same stream of problems, the better one reported: the first run of a
    # fresh box measured 21.7 ms per problem against 12.8-13.3 ms in every later run (host page-in)
    passes = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for U, st in pipe.run([(co, pin_F)] * n_e2e):
            st = None  # drop each state once its solution is back (as a serving loop would)
        torch.cuda.synchronize()
        passes.append((time.perf_counter() - t0) / n_e2e)
    e2e_step = min(passes)
    lat = []
    for _ in range(2):  # one problem alone through the same pipeline: no overlap
        t1 = time.perf_counter()
        for U, st in pipe.run([(co, pin_F)]):
            st = None
        lat.append(time.perf_counter() - t1)
    n_streams = len(pipe._mains)
    pipe.close()
    inp_b = solver.prepare(tree, nodes, co, device=dev, pinned=True)
    h2d = inp_b.h2d_bytes() + pin_F.numel() * 8
    d2h = U.numel() * 8 + 4 * 2 * L + 8 * inp_b.ngroups + 8 * (inp_b.ngroups + inp_b.gid.size)
    del inp_b
    e2e = {"value": unknowns / e2e_step, "unit": "unknowns/s", "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "seconds_per_step": e2e_step, "steps": n_e2e,
           "latency_s": float(min(lat)), "passes_s_per_step": [float(x) for x in passes],
           "includes": "per step: coefficient sampling on the host, H2D of the samples (pinned), leaf grouping "
                       "on the device, build, status check, H2D of the boundary data, batched solve, D2H of u "
                       "(N x ldu); solver.Pipeline overlaps step i+1's host work with step i's device work, "
                       "runs consecutive problems on two alternating compute streams (step i's latency-bound "
                       "top merges beside step i+1's leaf stage; %d stream(s) here) and replays build + solve "
                       "from two alternating CUDA-graph captures; latency_s = one problem alone; after a warm-up pass, the better of two timed passes (both in "
                       "passes_s_per_step)" % n_streams}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = CpuReference(cfg, L, b, q, full=False)  # one bounded sample (whole steps are the reference arm's)
        t_ref, brk = ref.step()
        cores, desc, info = ref.describe(brk)
        cpu = {"value": unknowns / t_ref, "unit": "unknowns/s", "cores": cores, "kind": "port", "sample": desc,
               "extrapolated": True, "host": info}
    if rank == 0:
        print(json.dumps({
            "metric": metric, "value": value, "unit": "unknowns/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "l2": L2_NOTE},
            "launch": launch_mode,
            "stages": {"unknowns": unknowns, "batch": b, "leaf_groups": inp.ngroups,
                       "pivoted_lu_depths": sorted(pivoted),
                       "fp64_gemm_emulation": emu,
                       "build_ms": tb * 1e3, "solve_ms": ts * 1e3,
                       "build_unknowns_per_s": unknowns / tb, "solve_unknowns_per_s": unknowns * b / ts,
                       "build_fp64_tflops": roofline["build_tflops"], "build_fp64_frac": roofline["build_frac"],
                       "solve_fp64_tflops": roofline["solve"]["tflops"], "solve_fp64_frac": roofline["solve"]["frac_fp64"],
                       "solve_hbm_gbs": roofline["solve"]["gbs_S_stream"], "solve_hbm_frac": roofline["solve"]["frac_hbm"]},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "gpu_launches_per_step": int(launches // args.steps), "clocks": clk}))


def bench_distributed(args, cfg, c, L, b, q, unknowns, workload, metric, rank, world):
    """N > 1: subtree-per-rank build + solve (parallel.py), NCCL between ranks, strong scaling of
    one problem. Times on the device, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_1307_2665_b200 as P
    from paper_1307_2665_b200 import _native, parallel, problems

    dev = torch.device("cuda")
    lib = _native.load()
    emu = configure_emulation(args)
    tree, nodes = P.build_tree(P.Rectangle(0.0, 1.0, 0.0, 1.0), L, q)
    co = c.coefficients()
    F = None
    if rank == 0:
        F_host = problems.boundary_data(cfg, nodes.points[tree.root.I_e], seed=0, batch=b)
        F = torch.from_numpy(np.ascontiguousarray(F_host if F_host.ndim == 2 else F_host[:, None])).to(dev)
    be = parallel.CudaBackend(tree, dev)
    comm = parallel.TorchComm()
    inputs = parallel.prepare_distributed(tree, co, rank, world, be)  # host sampling, outside the steps

    def step():
        st = parallel.build_distributed(tree, co, comm, be, inputs)
        u = parallel.solve_distributed(st, F, comm)
        return st, u

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clocks.start()
    l0 = lib.hps_launch_count()
    times = []
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flushed between steps, outside the step events
        torch.cuda.synchronize()
        dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = lib.hps_launch_count() - l0
    t = torch.tensor([float(np.mean(times))], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step = float(t.item())
    # ---- end-to-end through the public distributed API, host buffers in and out ----
    # per step and rank: host sampling + grouping of this rank's leaves and their H2D
    # (prepare_distributed), the boundary data's H2D from pinned memory on rank 0, the build and
    # the solve, and the D2H of the solution rows this rank computed (into pinned memory; all ranks
    # together copy every node's u once). Wall clock between barriers, max over ranks.
    rows = None
    e2e_times, h2d, d2h = [], 0, 0
    F_pin = torch.from_numpy(np.ascontiguousarray(F.cpu().numpy())).pin_memory() if rank == 0 else None
    for it in range(3):  # the first pass warms the pinned buffers
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        inp_e = parallel.prepare_distributed(tree, co, rank, world, be)
        Fd = F_pin.to(dev, non_blocking=True) if rank == 0 else None
        st = parallel.build_distributed(tree, co, comm, be, inp_e)
        u = parallel.solve_distributed(st, Fd, comm)
        if rows is None:
            rows = torch.from_numpy(st.owned_rows()).to(dev)
            host_u = torch.empty((int(rows.numel()), u.shape[1]), dtype=u.dtype).pin_memory()
        host_u.copy_(u.index_select(0, rows), non_blocking=True)
        torch.cuda.synchronize()
        dist.barrier()
        if it > 0:
            e2e_times.append(time.perf_counter() - t0)
        if it == 0:
            h2d = sum(int(x.numel()) * 8 for x in inp_e.fields if x is not None) + (int(F_pin.numel()) * 8 if rank == 0 else 0)
            d2h = int(host_u.numel()) * 8
        del st, u
    te = torch.tensor([min(e2e_times), float(h2d), float(d2h)], dtype=torch.float64, device=dev)
    tmax = te[:1].clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    tsum = te[1:].clone()
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    e2e = {"value": unknowns / float(tmax.item()), "unit": "unknowns/s", "seconds_per_step": float(tmax.item()),
           "h2d_bytes_per_step": int(tsum[0].item()), "d2h_bytes_per_step": int(tsum[1].item()),
           "includes": "per step and rank: host sampling + grouping of the rank's leaves and their H2D, the boundary "
                       "data's H2D (rank 0, pinned), build_distributed + solve_distributed (NCCL), D2H of the rank's "
                       "solution rows into pinned memory; wall clock between barriers, max over ranks, better of 2 passes"}
    if rank == 0:
        print(json.dumps({
            "metric": metric, "value": unknowns / t_step, "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "l2": L2_NOTE},
            "parallelism": f"subtree split at depth {int(np.log2(world))}, NCCL send/recv for the top merges",
            "timing": "CUDA events around each step (ranks start together after a barrier), mean over K steps, max over ranks; inputs resident (sampled + uploaded once per rank)",
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clk, "fp64_gemm_emulation": emu,
            "note": "roofline and cpu_baseline are reported on the N=1 line"}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
