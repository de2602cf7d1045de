# r02i: one-pass norms, split ILP, gathered small-n3 solve: suite, solve depths, benches.
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "extreme" 2>&1 | grep -E "assert|Error|passed|failed" | head -5
timeout 1500 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
grep -E "FAILED" gpurun_out/pytest_gpu.log | head
timeout 600 python tools/solve_depths.py 5 2>&1 | tail -20
for c in 2 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'])"; done
timeout 1500 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], d['cpu_baseline']['value']); r=d['roofline']; print({k: r.get(k) for k in ('achieved','peak','frac','unit','stage_int8_tops')}); print(d['clocks'])"
tail -2 gpurun_out/bench_cfg5.err
