python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for c in 1 2 3; do for v in 0 128; do echo "== HPS_AHEAD_MIN_N3=$v cfg$c"; HPS_AHEAD_MIN_N3=$v python tools/stage_times.py $c 2>&1 | grep -E "device total"; done; done
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
