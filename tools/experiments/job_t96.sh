python -m pytest tests -m gpu -x -q -k "gemm or parity" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do for v in 0 1; do echo "== HPS_T96=$v cfg2"; HPS_T96=$v python tools/stage_times.py 2 2>&1 | grep -E "merge_d11 |device total"; done; done
for v in 0 1; do echo "== HPS_T96=$v cfg4"; HPS_T96=$v python tools/stage_times.py 4 2>&1 | grep -E "merge_d15 |device total"; done
