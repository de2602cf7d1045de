set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -rA -s -p no:cacheprovider -k "engines_bitwise" > gpurun_out/i8_tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/i8_tests.log
grep -E "tcgen05 |Error|error" gpurun_out/i8_tests.log | head -20
for s in "4096 4096 1024 64" "8192 8192 2048 16" "32768 32768 8192 1"; do
  for e in 0 2; do
    timeout 300 python tools/emu_profile.py $s 14 0 8192 $e 2>&1 | grep -v -i warn | head -4
  done
done
