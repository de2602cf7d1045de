python -m pytest tests -m gpu -x -q -k "leaf or golden or oracle or spec or general_q" > gpurun_out/pytest_asm.log 2>&1; tail -2 gpurun_out/pytest_asm.log
for i in 1 2; do for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do echo "== $lib cfg2"; HPS_LIB=$PWD/$lib python tools/stage_times.py 2 2>&1 | grep -E "leaf "; done; done
for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do echo "== $lib cfg4"; HPS_LIB=$PWD/$lib python tools/stage_times.py 4 2>&1 | grep -E "leaf "; done
python tools/leaf3_phase_profile.py 2 | head -3
