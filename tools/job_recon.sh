set -u
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "emulated" 2>&1 | tail -1
for s in "4096 4096 1024 64" "32768 32768 8192 1" "3072 3072 512 128"; do
  timeout 300 python tools/emu_profile.py $s 14 0 8192 0 2>&1 | grep -v -i warn | head -4
done
