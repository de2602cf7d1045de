HPS_LEAF_V4=1 timeout 900 python -m pytest tests -m gpu -x -q -k "leaf or golden or oracle or spec" > gpurun_out/pytest_v4.log 2>&1; tail -3 gpurun_out/pytest_v4.log
for i in 1 2; do for v in 0 1; do echo "== HPS_LEAF_V4=$v cfg2"; HPS_LEAF_V4=$v python tools/stage_times.py 2 2>&1 | grep -E "leaf |device total"; done; done
for v in 0 1; do echo "== HPS_LEAF_V4=$v cfg4"; HPS_LEAF_V4=$v python tools/stage_times.py 4 2>&1 | grep -E "leaf |device total"; done
HPS_LEAF_V4=1 python tools/leaf3_phase_profile.py 2
