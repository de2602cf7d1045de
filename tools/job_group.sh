set -u
for g in 8 16 32 64 0; do
  timeout 300 python tools/emu_profile.py 32768 32768 8192 1 14 0 8192 0 $g 2>&1 | grep -v -i warn | head -2
done
for g in 8 32 0; do
  timeout 300 python tools/emu_profile.py 8192 8192 2048 16 14 0 8192 0 $g 2>&1 | grep -v -i warn | head -2
done
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "emulated" 2>&1 | tail -1
for es in 0 1; do
timeout 1200 python bench.py --no-cpu-baseline --emu-solve $es > gpurun_out/bench_cfg5_s$es.json 2> gpurun_out/bench_cfg5_s$es.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5_s$es.json').read().strip().splitlines()[-1]);print(5, 'solve-emu', $es, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], {k: round(v, 2) for k, v in d['roofline']['stage_ms'].items()})"
done
