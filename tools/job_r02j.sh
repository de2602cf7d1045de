set -u
mkdir -p gpurun_out
for mk in 1024 512; do
timeout 1500 python bench.py --no-cpu-baseline --emu-min-k $mk > gpurun_out/bench_cfg5_k$mk.json 2> gpurun_out/bench_cfg5_k$mk.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5_k$mk.json').read().strip().splitlines()[-1]);print(5, $mk, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], {k: round(v, 1) for k, v in d['roofline']['stage_ms'].items()}); r=d['roofline']; print({k: r.get(k) for k in ('achieved','peak','frac')}, d['clocks'])"
done
for c in 3 4; do for mk in 1024 512; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --emu-min-k $mk > gpurun_out/bench_cfg${c}_k$mk.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg${c}_k$mk.json').read().strip().splitlines()[-1]);print($c, $mk, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'])"; done; done
