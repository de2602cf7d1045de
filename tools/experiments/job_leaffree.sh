for i in 1 2; do for f in 0 4 8 16 32; do echo "free=$f"; HPS_LEAF_FREE_SMS=$f python tools/pipeline_probe.py 2 16 g 2>&1 | grep "jobs:" | head -1; done; done
for f in 0 8; do echo "device free=$f"; HPS_LEAF_FREE_SMS=$f python tools/stage_times.py 2 2>&1 | grep -E "leaf |device total"; done
