# Emulated block-inverse GEMMs + emulated batched solve: GPU suite, configs 3-5, min-K sweep on cfg 5.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
grep -E "diff .* gate|exact solution|FAILED" gpurun_out/pytest_gpu.log | head -40
for c in 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], {k: round(v, 2) for k, v in d['roofline']['stage_ms'].items()})"; done
for mk in 1024 512 256; do
timeout 1200 python bench.py --no-cpu-baseline --emu-min-k $mk > gpurun_out/bench_cfg5_k$mk.json 2> gpurun_out/bench_cfg5_k$mk.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5_k$mk.json').read().strip().splitlines()[-1]);print(5, $mk, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], {k: round(v, 2) for k, v in d['roofline']['stage_ms'].items()}); r=d['roofline']; print({k: r[k] for k in ('achieved','peak','frac','unit')})"
tail -1 gpurun_out/bench_cfg5_k$mk.err
done
