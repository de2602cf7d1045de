# Modular emulation on the tcgen05 kernel by default: full GPU suite, smoke, configs 2-5 benches.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
grep -E "diff .* gate|exact solution|FAILED" gpurun_out/pytest_gpu.log | head -40
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
for c in 2 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], {k: round(v, 2) for k, v in d['roofline']['stage_ms'].items()})"; done
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], {k: round(v, 2) for k, v in d['roofline']['stage_ms'].items()}); r=d['roofline']; print({k: r[k] for k in ('achieved','peak','frac','unit')})"
tail -2 gpurun_out/bench_cfg5.err
