set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
timeout 600 python tools/solve_depths.py 5 2>&1 | tail -19
set -u
for e in 0 2; do
for s in "32768 32768 8192 1" "8192 8192 2048 16" "3072 3072 512 128"; do
  timeout 300 python tools/emu_profile.py $s 14 0 8192 $e 2>&1 | grep -v -i warn | head -3
done; done
timeout 300 python tools/emu_profile.py 3072 3072 512 128 0 0 2>&1 | grep -v -i warn | head -2
