python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
bash tools/ab2.sh > gpurun_out/ab.txt 2>&1
python tools/leaf3_phase_profile.py 2 > gpurun_out/leaf3_phases.txt 2>&1
for c in 3 5; do for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do echo "== $lib cfg$c"; HPS_LIB=$PWD/$lib timeout 300 python tools/stage_times.py $c 2>&1 | grep -E "leaf |device total"; done; done >> gpurun_out/ab.txt 2>&1
