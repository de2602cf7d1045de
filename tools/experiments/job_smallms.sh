python -m pytest tests -m gpu -x -q -k "gemm or parity or solve" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do for v in 0 1; do echo "== HPS_SMALLM_S=$v cfg2"; HPS_SMALLM_S=$v python tools/stage_times.py 2 2>&1 | grep -E "merge_d(11|10|9) |device total"; done; done
for v in 0 1; do echo "== HPS_SMALLM_S=$v cfg4"; HPS_SMALLM_S=$v python tools/stage_times.py 4 2>&1 | grep -E "merge_d(15|14|13) |device total"; done
