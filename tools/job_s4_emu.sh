set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "emu or i8gemm" > gpurun_out/s4_emu_tests.log 2>&1; tail -3 gpurun_out/s4_emu_tests.log
python tools/emu_profile.py 16384 16384 4096 1 14 0 8192 0 0 1 2>&1 | grep -v -i Warn | head -8
timeout 900 $NCU --set full --import-source on --clock-control none -k "regex:k_crt_split" -c 2 -o gpurun_out/s4_split -f python tools/emu_profile.py 16384 16384 4096 1 14 0 8192 0 0 1 > gpurun_out/s4_ncu_split.log 2>&1; tail -1 gpurun_out/s4_ncu_split.log
