"""Write the leaf kernel's ncu --set full summary as JSON (the traffic source of bench.py's roofline).
Usage: python tools/ncu_leaf_json.py report.ncu-rep out.json "capture command" """
import csv, json, subprocess, sys
rep, out_path, cmd = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units, r = rows[0], rows[1], rows[2]
d = dict(zip(h, r)); u = dict(zip(h, units))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size"]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def bytes_of(k):
    return float(d[k].replace(",", "")) * scale.get(u[k], 1.0)
ms = float(d["gpu__time_duration.sum"]) * {"msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6}.get(u["gpu__time_duration.sum"], 1.0)
rd, wr = bytes_of("dram__bytes_read.sum"), bytes_of("dram__bytes_write.sum")
ngroups = 4096
res = {"kernel": "hps::k_leaf16v3", "workload": "cfg2_var_diffusion_L6_p16_b64", "groups_per_launch": ngroups,
       "capture": cmd, "gpu_time_ms": ms, "dram_read_bytes": rd, "dram_write_bytes": wr,
       "dram_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": ngroups * 139000.0,
       "raw": {k: d.get(k) + " " + u.get(k, "") for k in keys if k in d}}
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res, indent=1))
