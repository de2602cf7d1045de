python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do for v in 0 1; do echo "== HPS_SPLITK_FIXUP=$v cfg2"; HPS_SPLITK_FIXUP=$v python tools/stage_times.py 2 2>&1 | grep -E "merge_d[0-4] |device total|solve"; done; done
for v in 0 1; do echo "== HPS_SPLITK_FIXUP=$v cfg3"; HPS_SPLITK_FIXUP=$v python tools/stage_times.py 3 2>&1 | grep -E "device total|solve"; done
for v in 0 1; do echo "== HPS_SPLITK_FIXUP=$v cfg5"; HPS_SPLITK_FIXUP=$v timeout 600 python tools/stage_times.py 5 2>&1 | grep -E "device total|solve"; done
