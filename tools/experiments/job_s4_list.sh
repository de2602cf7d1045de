set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python tools/one_build.py 5 > gpurun_out/ncu_list.log 2>&1; tail -1 gpurun_out/ncu_list.log
python tools/one_build_launches.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5.md 2>&1; head -30 gpurun_out/launches_cfg5.md
