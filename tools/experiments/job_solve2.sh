python -m pytest tests -m gpu -x -q -k "solve or parity or exact or full_size or post" > gpurun_out/pytest_solve.log 2>&1; tail -2 gpurun_out/pytest_solve.log
for i in 1 2; do for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do for c in 1 3 4; do echo "== $lib cfg$c"; HPS_LIB=$PWD/$lib python tools/stage_times.py $c 2>&1 | grep -E "solve"; done; done; done
