"""Group an ncu launch list of ONE build (tools/one_build.py under ncu) by kernel kind and by merge
depth, in launch order (dev tool). Usage: python tools/one_build_launches.py launches.csv"""
import collections, sys
sys.path.insert(0, ".")
from tools.launch_summary import load
data = load(sys.argv[1])
# split into builds at each leaf-stage launch; keep the last complete build
starts = [i for i, d in enumerate(data) if "k_leaf" in d[0] and "hash" not in d[0] and "verify" not in d[0]]
seg = data[starts[-1]:] if starts else data
by_kind = collections.defaultdict(float)
depth = -1
by_depth = collections.defaultdict(float)
by_dk = collections.defaultdict(float)
for name, grid, block, us in seg:
    short = name.split("(")[0].replace("void ", "").replace("hps::", "")
    if "k_gather_xr" in short:
        depth += 1
    key = short[:48]
    by_kind[key] += us
    by_depth[depth] += us
    by_dk[(depth, key[:28])] += us
tot = sum(by_kind.values())
print(f"one build: {tot/1e3:.3f} ms serialized over {len(seg)} launches")
for k, v in sorted(by_kind.items(), key=lambda x: -x[1]):
    print(f"  {v/1e3:8.3f} ms {100*v/tot:5.1f}%  {k}")
print("by merge step (launch order; -1 = leaf stage):")
for d, v in sorted(by_depth.items()):
    parts = ", ".join(f"{k} {u:.0f}us" for (dd, k), u in sorted(by_dk.items(), key=lambda x: -x[1]) if dd == d)
    print(f"  step {d:3d}: {v/1e3:8.3f} ms   {parts}")
