"""Predicted N-GPU build time of config 5 (L = 9) for the two top-merge modes of parallel.py, from
the measured single-GPU stage times (profiles/bench_cfg5_*.json) and stated link / pipe rates.

    python tools/multigpu_model.py [profiles/bench_cfg5_r02k.json]

Model:
* ranks own the subtrees at depth s = log2 N: the leaf stage (one coefficient group at config 5) and
  every depth >= s run on each rank with 1/N of the boxes, at the measured single-GPU stage time / N;
* top depth d < s, group of P = 2^(s-d) ranks:
  - "owner": child b's DtN map moves to the owner (m^2 doubles), which runs the whole measured stage;
  - "panels": the same move; the owner forms and inverts the interface (2 n3^3 flop); it broadcasts
    the inverse and C to its group (one NCCL broadcast each) and sends a column panel of R to each of
    the P - 1 other ranks; every rank solves its panel
    (2 n3^2 ne / P flop) and forms its T panel (2 ne n3 ne / P flop); the T and S panels return; the
    owner assembles T = blkdiag + panels (3 ne^2 doubles of HBM traffic).
Rates: FP64 GEMM at the measured 33.8 TF/s of the top merges (config 5 depth 0), the interface
inverse at 20 TF/s, NVLink 5 point-to-point at LINK_GBS per direction per GPU (NCCL send/recv of
large buffers; nominal 900 GB/s), HBM 6.5 TB/s."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
from paper_1307_2665_b200 import work as W  # noqa: E402

GEMM_TF = 33.8e12
INV_TF = 20e12
LINK_GBS = 600e9
HBM = 6.5e12


def model(stage_ms, L=9, q=16, world=8, gemm_tf=None, inv_tf=None):
    GEMM_TF_ = gemm_tf or GEMM_TF
    INV_TF_ = inv_tf or INV_TF
    s = world.bit_length() - 1
    t_local = stage_ms["leaf"] / 1e3 + sum(stage_ms[f"merge_d{d}"] / 1e3 for d in range(s, 2 * L)) / world
    rows = []
    t_owner = t_panels = t_local
    for d in range(s - 1, -1, -1):
        n3, ne = W.depth_sizes(L, q, d)
        m = ne // 2 + n3
        P = 1 << (s - d)
        move = 8.0 * m * m / LINK_GBS
        # the measured stage merges all 2^d boxes of the depth batched; each owner merges one
        own = move + stage_ms[f"merge_d{d}"] / 1e3 / (1 << d)
        inv = 2.0 * n3 ** 3 / INV_TF_
        gather = 8.0 * (n3 * n3 + 2 * n3 * ne) * 2 / HBM
        # the factored interface and C go to the group by one NCCL broadcast each (pipelined ring:
        # about one copy per link), the R column panels point to point
        out = 8.0 * (n3 * n3 + ne * n3) / LINK_GBS + 8.0 * (P - 1) * (n3 * ne / P) / LINK_GBS
        compute = (2.0 * n3 * n3 * ne + 2.0 * ne * n3 * ne) / P / GEMM_TF_
        back = 8.0 * (P - 1) * (ne * ne / P + n3 * ne / P) / LINK_GBS
        assemble = 8.0 * 3 * ne * ne / HBM
        pan = move + gather + inv + out + compute + back + assemble
        t_owner += own
        t_panels += pan
        rows.append({"depth": d, "P": P, "n3": n3, "ne": ne, "owner_s": own, "panels_s": pan,
                     "panels_parts_s": {"move_child_T": move, "gather": gather, "inverse": inv, "send": out,
                                        "solve_and_T_GEMM": compute, "return": back, "assemble": assemble}})
    t1 = stage_ms["leaf"] / 1e3 + sum(v / 1e3 for k, v in stage_ms.items() if k.startswith("merge_d"))
    return {"world": world, "t_1gpu_build_s": t1, "t_local_s": t_local, "owner": t_owner, "panels": t_panels,
            "speedup_owner": t1 / t_owner, "speedup_panels": t1 / t_panels, "top_depths": rows,
            "rates": {"gemm_tflops": GEMM_TF_ / 1e12, "inverse_tflops": INV_TF_ / 1e12, "link_gbs": LINK_GBS / 1e9,
                      "hbm_tbs": HBM / 1e12}}


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "..", "profiles", "bench_cfg5_r02a.json")
    d = json.loads(open(path).read().strip().splitlines()[-1])
    stage_ms = d["roofline"]["stage_ms"]
    # with the FP64 emulation on, the top merges' GEMMs run at the measured FP64-equivalent rate of the
    # dominant (depth-0) stage, and the interface inverse's GEMMs at about half of it
    fe = d["roofline"].get("fp64_equivalent", {}).get("achieved_tflops")
    gemm_tf = fe * 1e12 if fe else None
    inv_tf = 0.5 * fe * 1e12 if fe else None
    out = {"source": os.path.basename(path), "gemm_tflops_used": (gemm_tf or GEMM_TF) / 1e12,
           "models": [model(stage_ms, world=w, gemm_tf=gemm_tf, inv_tf=inv_tf) for w in (2, 4, 8)]}
    for r in out["models"]:
        print(f"N={r['world']}: 1 GPU {r['t_1gpu_build_s']*1e3:7.1f} ms | owner-computes {r['owner']*1e3:7.1f} ms "
              f"({r['speedup_owner']:.2f}x) | panels {r['panels']*1e3:7.1f} ms ({r['speedup_panels']:.2f}x)")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
