set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec.py tests/test_gpu_baseline_sizes.py tests/test_gpu_multigpu.py -m gpu -q > gpurun_out/s4_tests.log 2>&1; tail -2 gpurun_out/s4_tests.log
run() { timeout 300 python bench.py --config $1 --no-cpu-baseline > gpurun_out/s4_ab.json 2> gpurun_out/s4_ab.err; python -c "
import json,sys; d=json.loads(open('gpurun_out/s4_ab.json').read().strip().splitlines()[-1]); st=d['stages']; print($1, round(d['ms_per_step'],3), round(st['build_ms'],3), round(st['solve_ms'],3), round(d['e2e']['seconds_per_step']*1e3,2))"; }
run 5
run 2
