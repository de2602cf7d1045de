set -u
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "i8gemm or engines" 2>&1 | tail -1
for e in 2 0; do
timeout 300 python tools/emu_profile.py 32768 32768 8192 1 14 0 8192 $e 2>&1 | grep -v -i warn | head -2 | tail -1
timeout 300 python tools/emu_profile.py 8192 8192 2048 16 14 0 8192 $e 2>&1 | grep -v -i warn | head -2 | tail -1
done
