set -u
for g in 1 2 4 8 32 64 128; do
  timeout 300 python tools/emu_profile.py 32768 32768 8192 1 14 0 8192 2 $g 2>&1 | grep -v -i warn | head -2 | tail -1
done
timeout 300 python tools/emu_profile.py 32768 32768 8192 1 14 0 8192 0 0 2>&1 | grep -v -i warn | head -2 | tail -1
