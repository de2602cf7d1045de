"""Attribute ncu SASS-level warp-stall samples to source lines (dev tool).
Usage: python tools/ncu_lines.py report.ncu-rep kernel_regex cubin [top]
The cubin must be compiled with the same flags as the profiled library (-lineinfo)."""
import csv, collections, re, subprocess, sys
rep, kre, cubin = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") or c.startswith("Warp Stall Sampling (All")]
iall = h.index("Warp Stall Sampling (All Samples)")
sass = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout.split("\n")
off2 = {}; cur = None; fn = None
for l in sass:
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m: fn = m.group(1)
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2)))
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and fn and re.search(kre, fn): off2[int(m.group(1), 16)] = cur
base = int(data[0][ia], 16)
tot = collections.Counter(); reasons = collections.defaultdict(collections.Counter)
for r in data:
    key = off2.get(int(r[ia], 16) - base)
    tot[key] += int(r[iall])
    for i in stall_cols:
        if i != iall and r[i] not in ("", "0"):
            try: reasons[key][h[i]] += int(r[i])
            except ValueError: pass
S = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
    rs = ", ".join(f"{n}:{c}" for n, c in reasons[k].most_common(3))
    print(f"{str(k):28s} {v:7d} {100*v/S:5.1f}%  {rs}")
