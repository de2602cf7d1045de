# Full ncu capture of the largest single-RHS solve launch of one config-4 build + solve (HBM-bound).
set -u
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_solve --csv --log-file gpurun_out/solve_list.csv python tools/one_build.py 4 > /dev/null 2>&1
SKIP=$(python - <<'PY'
import sys; sys.path.insert(0, ".")
from tools.launch_summary import load
d = load("gpurun_out/solve_list.csv")
print(max(range(len(d)), key=lambda k: d[k][3]))
PY
)
echo "skip=$SKIP"
python - <<'PY'
import sys; sys.path.insert(0, ".")
from tools.launch_summary import load
d = load("gpurun_out/solve_list.csv")
for n, g, b, us in d: print(n.split("(")[0][:40], g, us)
PY
ncu --set full --clock-control none -k regex:k_solve --launch-skip $SKIP -c 1 -o gpurun_out/prof_solve_cfg4 python tools/one_build.py 4 > gpurun_out/ncu_solve.log 2>&1
tail -1 gpurun_out/ncu_solve.log
