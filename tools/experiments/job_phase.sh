set -u
python tools/leaf3_phase_profile.py 2 > gpurun_out/leaf3_phases_cfg2.txt 2>&1
python tools/stage_times.py 2 > gpurun_out/stage_cfg2.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_one_build.csv python tools/one_build.py 2 > gpurun_out/ncu_one.log 2>&1
python tools/one_build_launches.py gpurun_out/launches_one_build.csv > gpurun_out/one_build_summary.txt 2>&1
echo done
