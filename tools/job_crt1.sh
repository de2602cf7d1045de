# Modular (CRT) FP64 emulation: accuracy tests, then the full GPU suite and configs 3 / 5 benches.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -rA -s -p no:cacheprovider -k emulated > gpurun_out/crt_tests.log 2>&1; tail -3 gpurun_out/crt_tests.log
grep -E "emulated \(|Error|error" gpurun_out/crt_tests.log | head -30
timeout 1500 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
grep -E "diff .* gate|exact solution|FAILED" gpurun_out/pytest_gpu.log | head -40
for c in 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['roofline']['stage_ms'])"; done
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['roofline']['stage_ms'])"
tail -2 gpurun_out/bench_cfg5.err
