set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "emulated" 2>&1 | tail -1
for s in "4096 4096 1024 64" "3072 3072 512 128" "32768 32768 8192 1"; do
  timeout 300 python tools/emu_profile.py $s 14 0 8192 0 2>&1 | grep -v -i warn | head -7
done
timeout 300 python tools/emu_profile.py 3072 3072 512 128 0 0 2>&1 | grep -v -i warn | head -3
for mk in 1024 512; do
timeout 1200 python bench.py --no-cpu-baseline --emu-min-k $mk > gpurun_out/bench_cfg5_k$mk.json 2> gpurun_out/bench_cfg5_k$mk.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5_k$mk.json').read().strip().splitlines()[-1]);print(5, $mk, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], {k: round(v, 2) for k, v in d['roofline']['stage_ms'].items()}); r=d['roofline']; print({k: r[k] for k in ('achieved','peak','frac','unit')}, d['clocks'])"
done
