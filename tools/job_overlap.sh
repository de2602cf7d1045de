set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "emulated or i8gemm" 2>&1 | tail -1
for s in "4096 4096 1024 64" "32768 32768 8192 1" "8192 8192 2048 16"; do
  timeout 300 python tools/emu_profile.py $s 14 0 8192 0 2>&1 | grep -v -i warn | head -1
done
for ov in 1 0; do
python - $ov <<'PY'
import sys; sys.argv=[sys.argv[0]]
PY
done
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], {k: round(v, 1) for k, v in d['roofline']['stage_ms'].items()}); print(d['clocks'])"
for c in 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'])"; done
