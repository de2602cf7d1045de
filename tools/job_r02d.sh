# Round 2: FP64 GEMM emulation on by default -- full GPU suite, smoke, bench lines of configs 2-5.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
grep -E "diff .* gate|exact solution|FAILED|emulated \(" gpurun_out/pytest_gpu.log | head -60
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
for c in 2 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d['e2e']['seconds_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'])"; done
timeout 1200 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['e2e'], d['stages'], d['roofline']['frac'])"
tail -2 gpurun_out/bench_cfg5.err
