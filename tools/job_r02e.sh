# Round 2 session 2 re-entry: state check -- GPU suite, smoke, default bench (cfg5), int8 probe.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python tools/int8_probe.py > gpurun_out/int8_probe.txt 2>&1; cat gpurun_out/int8_probe.txt
timeout 1200 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
tail -c 600 gpurun_out/bench_cfg5.json; tail -2 gpurun_out/bench_cfg5.err
