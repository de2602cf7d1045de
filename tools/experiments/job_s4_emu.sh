set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "emu or i8gemm" > gpurun_out/s4_emu_tests.log 2>&1; tail -2 gpurun_out/s4_emu_tests.log
python tools/emu_profile.py 16384 16384 4096 1 14 0 8192 0 0 1 2>&1 | grep -v -i Warn | head -8
python tools/emu_profile.py 4096 24576 4096 2 14 0 8192 0 0 1 2>&1 | grep -v -i Warn | head -8
