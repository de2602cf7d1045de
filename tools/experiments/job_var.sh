for i in 1 2 3 4 5 6; do python tools/stage_times.py 2 2>&1 | grep -E "device total|leaf "; done
