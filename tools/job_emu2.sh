set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rA -k "emulated" > gpurun_out/pytest_emu.log 2>&1; tail -2 gpurun_out/pytest_emu.log
for e in 0 8; do
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --emu-slices $e > gpurun_out/bench_cfg5_emu$e.json 2> gpurun_out/bench_cfg5_emu$e.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5_emu$e.json').read().strip().splitlines()[-1]);print('emu $e', d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], {k: round(v,1) for k,v in d['roofline']['stage_ms'].items()})"
tail -2 gpurun_out/bench_cfg5_emu$e.err
done
for c in 3; do for e in 0 8; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --emu-slices $e > gpurun_out/bench_cfg${c}_emu$e.json 2> gpurun_out/bench_cfg${c}_emu$e.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg${c}_emu$e.json').read().strip().splitlines()[-1]);print('cfg$c emu $e', d['ms_per_step'], d['stages']['build_ms'])"
done; done
