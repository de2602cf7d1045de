"""The int8 kernel's ncu capture as the JSON bench.py reads its DRAM traffic from (dev tool).
Usage: python tools/ncu_i8_json.py report.ncu-rep M nc K moduli "capture note" > profiles/i8gemm_cfg5_d0_ncu_<tag>.json"""
import csv
import json
import subprocess
import sys

path, M, nc, K, nmod, note = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
d = {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def num(key, scale):
    v, u = d[key]
    return float(v) * scale.get(u, 1.0)


byte_units = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
time_units = {"ms": 1.0, "us": 1e-3, "s": 1e3, "ns": 1e-6}
rd, wr = num("dram__bytes_read.sum", byte_units), num("dram__bytes_write.sum", byte_units)
ms = num("gpu__time_duration.sum", time_units)
ops = 2.0 * M * nc * K * nmod
alg = float(nmod) * (M * K + nc * K + M * nc)
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
print(json.dumps({
    "kernel": f"hps::i8::k_i8gemm_mod (tcgen05.mma.kind::i8; merge depth 0 T GEMM residue products, one output column panel: "
              f"{M} x {nc} x {K}, {nmod} moduli; 8 epilogue warps)",
    "workload": "cfg5_conv_diffusion_b1000_L9_p16_b256",
    "stage": "merge_d0_i8",
    "capture": note,
    "gpu_time_ms": ms,
    "dram_read_bytes": rd,
    "dram_write_bytes": wr,
    "dram_bytes_per_launch": rd + wr,
    "algorithmic_bytes_per_launch": alg,
    "algorithmic_int8_ops_per_launch": ops,
    "achieved_tops_under_ncu": ops / ms / 1e9,
    "raw": {k: " ".join(d[k]) for k in keys if k in d},
}, indent=1))
