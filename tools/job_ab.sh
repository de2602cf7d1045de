python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
bash tools/ab2.sh > gpurun_out/ab.txt 2>&1
python tools/leaf3_phase_profile.py 2 > gpurun_out/leaf3_phases.txt 2>&1
