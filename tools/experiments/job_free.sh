python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do for v in 0 4 8 16; do echo "== HPS_AHEAD_FREE_SMS=$v cfg2"; HPS_AHEAD_FREE_SMS=$v python tools/stage_times.py 2 2>&1 | grep -E "merge_d[0-5] |device total"; done; done
for v in 0 8 16; do echo "== HPS_AHEAD_FREE_SMS=$v cfg3"; HPS_AHEAD_FREE_SMS=$v python tools/stage_times.py 3 2>&1 | grep -E "device total"; done
HPS_AHEAD_FREE_SMS=8 python tools/ahead_probe.py 2
