python -m pytest tests -m gpu -x -q -k "gemm or parity" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in 0 16 24; do echo "== GROUP_M=$v"; HPS_GEMM_GROUP_M=$v python tools/bench_inverse.py 2>&1 | grep -E "gemm (4096x4096|8192x8192|3072x3072|1024x4096)"; done
for v in 0 16; do echo "== GROUP_M=$v cfg2"; HPS_GEMM_GROUP_M=$v python tools/stage_times.py 2 2>&1 | grep -E "device total"; done
for v in 0 16 24; do echo "== GROUP_M=$v cfg3"; HPS_GEMM_GROUP_M=$v python tools/stage_times.py 3 2>&1 | grep -E "merge_d0 |merge_d1 |device total"; done
for v in 0 16; do echo "== GROUP_M=$v cfg4"; HPS_GEMM_GROUP_M=$v python tools/stage_times.py 4 2>&1 | grep -E "merge_d0 |device total"; done
for v in 0 16; do echo "== GROUP_M=$v cfg5"; HPS_GEMM_GROUP_M=$v timeout 900 python tools/stage_times.py 5 2>&1 | grep -E "merge_d0 |merge_d1 |device total"; done
HPS_GEMM_GROUP_M=16 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dgemm64 --launch-skip 258 -c 1 python tools/one_build.py 3 2>&1 | grep -E "dram__|duration" 
