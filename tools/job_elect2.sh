set -u
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "emulated or i8gemm" 2>&1 | tail -1
for e in 0 2; do timeout 300 python tools/emu_profile.py 32768 32768 8192 1 14 0 8192 $e 2>&1 | grep -v -i warn | head -2; done
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]);print(5, d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step']); r=d['roofline']; print({k: r.get(k) for k in ('achieved','peak','frac')}, d['clocks'])"
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none -k "regex:k_i8gemm" -c 1 -o gpurun_out/i8_elect -f python tools/emu_profile.py 32768 16384 8192 1 14 0 8192 0 > gpurun_out/ncu_elect.log 2>&1; tail -1 gpurun_out/ncu_elect.log
