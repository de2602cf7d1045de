for f in 0 8 16 24 32 48; do echo "free=$f"; HPS_LEAF_FREE_SMS=$f python tools/stage_times.py 2 2>&1 | grep -E "leaf "; done
for f in 0 16 32; do echo "cfg4 free=$f"; HPS_LEAF_FREE_SMS=$f python tools/stage_times.py 4 2>&1 | grep -E "leaf "; done
