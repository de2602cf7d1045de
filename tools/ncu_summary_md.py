"""Key metrics of one or more ncu reports as a markdown table (dev tool).
Usage: python tools/ncu_summary_md.py label=report.ncu-rep [...]"""
import csv
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active", "IMMA issue %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_size", "cluster"),
    ("launch__registers_per_thread", "regs/thread"),
]


def metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    return d


cols = []
for arg in sys.argv[1:]:
    label, path = arg.split("=", 1)
    cols.append((label, metrics(path)))
print("| metric | " + " | ".join(c[0] for c in cols) + " |")
print("|---|" + "---|" * len(cols))
print("| kernel | " + " | ".join(c[1].get("Kernel Name", ("?", ""))[0].split("(")[0][:60] for c in cols) + " |")
for key, name in METRICS:
    cells = []
    for _, d in cols:
        v, u = d.get(key, ("n/a", ""))
        cells.append(f"{v} {u}".strip())
    print(f"| {name} (`{key}`) | " + " | ".join(cells) + " |")
