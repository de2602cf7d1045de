set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -rA -s -p no:cacheprovider -k emulated > gpurun_out/crt_tests.log 2>&1; tail -2 gpurun_out/crt_tests.log
grep -E "emulated \(" gpurun_out/crt_tests.log | head -30
for s in "4096 4096 1024 64" "8192 8192 2048 16" "32768 32768 8192 1"; do
  timeout 300 python tools/emu_profile.py $s 14 0 2>&1 | grep -v Warn | head -9
done
