python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do echo "== $lib cfg2"; HPS_LIB=$PWD/$lib python tools/stage_times.py 2 2>&1 | grep -E "merge_d(11|10) |device total"; done; done
for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do echo "== $lib cfg4"; HPS_LIB=$PWD/$lib python tools/stage_times.py 4 2>&1 | grep -E "device total"; done
echo "== cfg5 new"; timeout 900 python tools/stage_times.py 5 2>&1 | grep -E "merge_d0 |device total"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gather|k_ahead" -c 60 --csv --log-file gpurun_out/launches_gather.csv python tools/one_build.py 2 > /dev/null 2>&1
