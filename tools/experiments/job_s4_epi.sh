set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "emu or i8gemm" > gpurun_out/s4_emu_tests.log 2>&1; tail -2 gpurun_out/s4_emu_tests.log
python tools/emu_profile.py 16384 16384 4096 1 2>&1 | grep -v -i warn | head -4
run() { timeout 300 python bench.py --config $1 --no-cpu-baseline > gpurun_out/s4_ab.json 2> gpurun_out/s4_ab.err; python -c "
import json,sys; d=json.loads(open('gpurun_out/s4_ab.json').read().strip().splitlines()[-1]); st=d['stages']; print($1, round(d['ms_per_step'],3), round(st['build_ms'],3), round(d['roofline']['achieved'],2))"; }
run 5
run 5
