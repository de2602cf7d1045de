# r02k: min-K 512 default, two-row reconstruction: emulation profiles, GPU suite, smoke, benches.
set -u
mkdir -p gpurun_out
for s in "4096 4096 1024 64" "32768 32768 8192 1" "3072 3072 512 128"; do
  timeout 300 python tools/emu_profile.py $s 14 0 8192 0 2>&1 | grep -v -i warn | head -3
done
timeout 1500 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
grep -E "diff .* gate|FAILED" gpurun_out/pytest_gpu.log | head -30
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for c in 2 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'])"; done
timeout 1500 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], d['cpu_baseline']['value']); r=d['roofline']; print({k: r.get(k) for k in ('achieved','peak','frac','unit','stage_int8_tops')}); print(d['clocks'])"
