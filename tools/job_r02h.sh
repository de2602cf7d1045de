# r02h: exact int8 kernel tests; cfg5 launch list of one build; ncu --set full of the depth-0 T-GEMM
# int8 kernel launch (the bench's dominant kernel); default bench line (cfg5) with the live kernel timing.
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "i8gemm or emulated" 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python tools/one_build.py 5 > gpurun_out/ncu_list.log 2>&1; tail -1 gpurun_out/ncu_list.log
python tools/one_build_launches.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5.md 2>&1; head -30 gpurun_out/launches_cfg5.md
SKIP=$(python - <<'PY'
import sys; sys.path.insert(0, ".")
from tools.launch_summary import load
d = load("gpurun_out/launches_cfg5.csv")
idx = [k for k in range(len(d)) if "k_i8gemm" in d[k][0]]
i = max(idx, key=lambda k: d[k][3])
print(idx.index(i))
PY
)
echo "skip=$SKIP"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_i8gemm --launch-skip $SKIP -c 1 -o gpurun_out/prof_i8gemm_cfg5_d0 -f python tools/one_build.py 5 > gpurun_out/ncu_i8_cfg5.log 2>&1
tail -2 gpurun_out/ncu_i8_cfg5.log
timeout 1500 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], d['cpu_baseline']['value']); r=d['roofline']; print({k: r.get(k) for k in ('achieved','peak','frac','unit','kernel','stage_int8_tops')}); print(r.get('kernel_live'))"
tail -2 gpurun_out/bench_cfg5.err
