# ncu --set full of the int8 panel products (tcgen05 single CTA / CTA pair / cuBLASLt) on one
# 32768 x 16384 x 8192 panel GEMM (merge depth 0's T GEMM shape, half width).
set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for e in 0 2 1; do
  timeout 600 $NCU --set full --import-source on --clock-control none -k "regex:k_i8gemm|cutlass" -c 1 \
    -o gpurun_out/i8_engine$e -f python tools/emu_profile.py 32768 16384 8192 1 14 0 8192 $e > gpurun_out/ncu_i8_e$e.log 2>&1
  tail -2 gpurun_out/ncu_i8_e$e.log
done
