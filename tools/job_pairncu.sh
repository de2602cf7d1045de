set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none -k "regex:k_i8gemm" -c 1 -o gpurun_out/i8_pair_now -f python tools/emu_profile.py 32768 16384 8192 1 14 0 8192 2 > gpurun_out/ncu_pair.log 2>&1; tail -1 gpurun_out/ncu_pair.log
timeout 600 $NCU --set full --clock-control none -k "regex:k_i8gemm" -c 1 -o gpurun_out/i8_single_now -f python tools/emu_profile.py 32768 16384 8192 1 14 0 8192 0 > gpurun_out/ncu_single.log 2>&1; tail -1 gpurun_out/ncu_single.log
