python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do echo "== $lib cfg2"; HPS_LIB=$PWD/$lib python tools/stage_times.py 2 2>&1 | grep -E "device total"; done; done
for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do echo "== $lib cfg3"; HPS_LIB=$PWD/$lib python tools/stage_times.py 3 2>&1 | grep -E "device total"; done
