set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/s4_gpu_tests.log 2>&1; tail -3 gpurun_out/s4_gpu_tests.log
for c in 5 3; do
python bench.py --config $c --no-cpu-baseline > gpurun_out/s4_bench$c.json 2> gpurun_out/s4_bench$c.err; python -c "
import json; d=json.loads(open('gpurun_out/s4_bench$c.json').read().strip().splitlines()[-1]); print($c, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], d['clocks'])"
done
