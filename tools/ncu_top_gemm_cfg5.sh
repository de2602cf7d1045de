# Full ncu capture of the largest dgemm64 launch of one config-5 build (L = 9): the depth-0 T GEMM
# T = blk + C S, 32768 x 32768 x 8192 (the dominant kernel of the default bench line).
set -u
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dgemm64 --csv --log-file gpurun_out/gemm_list_cfg5.csv python tools/one_build.py 5 > /dev/null 2>&1
SKIP=$(python - <<'PY'
import sys; sys.path.insert(0, ".")
from tools.launch_summary import load
d = load("gpurun_out/gemm_list_cfg5.csv")
i = max(range(len(d)), key=lambda k: d[k][3])
print(i)
PY
)
echo "skip=$SKIP"
ncu --set full --import-source on --clock-control none -k regex:dgemm64 --launch-skip $SKIP -c 1 -o gpurun_out/prof_dgemm64_cfg5_d0 python tools/one_build.py 5 > gpurun_out/ncu_gemm_cfg5.log 2>&1
tail -2 gpurun_out/ncu_gemm_cfg5.log
