nproc; cat /proc/cpuinfo | grep "model name" | head -1; uptime
python tools/e2e_breakdown.py 2 > gpurun_out/e2e_breakdown.txt 2>&1
python tools/pipeline_probe.py 2 16 g > gpurun_out/pipe_probe.txt 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_b.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_c.json 2>&1
bash tools/job_smallk.sh > gpurun_out/smallk.txt 2>&1
