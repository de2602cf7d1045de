set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/one_build.py 2 > /dev/null 2>&1
python tools/one_build_launches.py gpurun_out/launches_cfg2.csv 2>&1 | tail -16 | cut -c1-330
