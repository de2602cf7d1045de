# Launch list (ncu, time only) of one config-2 build + solve with the pivoted LU merges.
set -u
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_cfg2_lu.csv python tools/one_build.py 2 > gpurun_out/ncu_cfg2.log 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg2_lu.csv | head -30
python - <<'PY'
import sys; sys.path.insert(0, ".")
from tools.launch_summary import load
d = load("gpurun_out/launches_cfg2_lu.csv")
import collections
for name in ("k_lu_panel", "k_swap_trsm16", "k_strip_solve", "dgemm64", "k_permute_rows", "k_ipiv_to_perm", "k_nonfinite"):
    xs = [x[3] for x in d if name in x[0]]
    if xs:
        print(f"{name:16s} n={len(xs):5d} total {sum(xs)/1e3:8.3f} ms  mean {sum(xs)/len(xs):8.2f} us  max {max(xs):8.2f} us")
PY
