set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "emu or i8gemm" > gpurun_out/s4_emu_tests.log 2>&1; tail -3 gpurun_out/s4_emu_tests.log
python tools/emu_profile.py 16384 16384 4096 1 14 0 8192 0 2>&1 | grep -v -i Warn | head -8
python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s4_parity_tests.log 2>&1; tail -3 gpurun_out/s4_parity_tests.log
python bench.py --config 5 --no-cpu-baseline > gpurun_out/s4_bench5.json 2> gpurun_out/s4_bench5.err; python -c "
import json; d=json.loads(open('gpurun_out/s4_bench5.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['e2e']['seconds_per_step'], d['clocks'])"
