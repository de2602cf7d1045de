python -m pytest tests -m gpu -x -q -k "gemm or parity or solve" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do for v in 0 1; do echo "== HPS_SMALLM=$v cfg2"; HPS_SMALLM=$v python tools/stage_times.py 2 2>&1 | grep -E "solve|device total"; done; done
for v in 0 1; do echo "== HPS_SMALLM=$v cfg5"; HPS_SMALLM=$v timeout 600 python tools/stage_times.py 5 2>&1 | grep -E "solve"; done
for v in 0 1; do echo "== HPS_SMALLM=$v cfg3"; HPS_SMALLM=$v python tools/stage_times.py 3 2>&1 | grep -E "solve"; done
