# Final refresh of round 2, session 4: GPU suite, smoke, all configs, default bench line with CPU
# baseline, reference arm, launch list of one cfg5 build, ncu --set full of the bench's dominant
# kernel, the distributed leg at world size 1.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for c in 1 2 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]);print($c, round(d['ms_per_step'],2), round(d['stages']['build_ms'],2), round(d['stages']['solve_ms'],2), round(d['e2e']['seconds_per_step']*1e3,2))"; done
timeout 1500 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], d['cpu_baseline']['value']); r=d['roofline']; print({k: r.get(k) for k in ('achieved','peak','frac','unit','stage_int8_tops')}); print(d['clocks'])"
timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -c 400 gpurun_out/bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python tools/one_build.py 5 > gpurun_out/ncu_list.log 2>&1; tail -1 gpurun_out/ncu_list.log
python tools/one_build_launches.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5.md 2>&1; head -12 gpurun_out/launches_cfg5.md
SKIP=$(python - <<'PY'
import sys; sys.path.insert(0, ".")
from tools.launch_summary import load
d = load("gpurun_out/launches_cfg5.csv")
idx = [k for k in range(len(d)) if "k_i8gemm" in d[k][0]]
i = max(idx, key=lambda k: d[k][3])
print(idx.index(i))
PY
)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_i8gemm --launch-skip $SKIP -c 1 -o gpurun_out/prof_i8gemm_cfg5_d0 -f python tools/one_build.py 5 > gpurun_out/ncu_i8_cfg5.log 2>&1
tail -1 gpurun_out/ncu_i8_cfg5.log
timeout 900 ncu --set full --clock-control none -k "regex:k_crt_split|k_crt_accum|k_crt_col_scale|k_crt_row_scale" -c 5 -o gpurun_out/prof_emu_aux -f python tools/emu_profile.py 16384 16384 4096 1 > gpurun_out/ncu_aux.log 2>&1; tail -1 gpurun_out/ncu_aux.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --force-distributed --no-cpu-baseline > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; tail -c 300 gpurun_out/bench_dist1.json
