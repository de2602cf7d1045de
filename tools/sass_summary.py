"""Per-kernel SASS evidence of the product library (dev tool): counts of the tensor / TMA / TMEM /
barrier mnemonics in every kernel of libhps_b200.so (cuobjdump -sass), as a markdown table.
Usage: python tools/sass_summary.py [path/to/libhps_b200.so] > profiles/sass_summary_<tag>.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1307_2665_b200/libhps_b200.so"
MN = ["DMMA", "UTCIMMA", "IMMA", "UTMALDG", "UTCBAR", "LDTM", "SYNCS", "REDUX", "LDGSTS", "DFMA", "SHFL"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
names = subprocess.run(["c++filt"], input="\n".join(re.findall(r"Function : (\S+)", sass)), capture_output=True, text=True).stdout.splitlines()
res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
regs = dict(re.findall(r"Function (\S+):\n\s+REG:(\d+)", res))
kern, cur, total = collections.OrderedDict(), None, collections.Counter()
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kern[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(1)
        kern[cur]["_n"] += 1
        for k in MN:
            if op == k or op.startswith(k + "."):
                kern[cur][k] += 1
print("# SASS evidence per kernel of libhps_b200.so (sm_100a; cuobjdump -sass; tools/sass_summary.py)")
print()
print("Static instruction counts. DMMA = FP64 tensor (mma.sync.m8n8k4.f64), UTCIMMA = tcgen05.mma.kind::i8, UTMALDG = TMA")
print("tensor load, LDTM = tcgen05.ld, SYNCS = mbarrier operations, UTCBAR = tcgen05.commit, IMMA = legacy int8")
print("mma.sync (the residue kernels), LDGSTS = cp.async, REDUX = warp reductions (pivot search).")
print()
print("| kernel | regs | instructions | " + " | ".join(MN) + " |")
print("|---|---|---|" + "---|" * len(MN))
for (mangled, c), name in zip(kern.items(), names):
    short = re.sub(r"\(.*", "", name).replace("void ", "").replace("hps::", "")
    if not any(c[k] for k in MN):
        continue
    print(f"| `{short[:70]}` | {regs.get(mangled, '?')} | {c['_n']} | " + " | ".join(str(c[k]) if c[k] else "" for k in MN) + " |")
