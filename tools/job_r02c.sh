# Round 2: residual-checked block inverse (default) + pivoted LU fallback; tests, bench lines, LU launch list.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_multigpu.py -q -rA > gpurun_out/pytest_lu.log 2>&1; tail -12 gpurun_out/pytest_lu.log
timeout 1200 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
grep -E "diff .* gate|exact solution|FAILED" gpurun_out/pytest_gpu.log | head -40
for c in 2 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d['e2e']['seconds_per_step'], d['stages']['pivoted_lu_depths'], d['roofline']['stage_ms'])"; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['stages']['build_ms'], d['roofline']['stage_ms'])"
tail -3 gpurun_out/bench_cfg5.err
