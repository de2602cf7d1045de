set -u
mkdir -p gpurun_out
timeout 300 python tools/emu_profile.py 4096 4096 1024 64 14 0 8192 0 2>&1 | grep -v -i warn | head -3
timeout 900 python bench.py --config 2 --force-distributed --steps 3 --warmup 2 > gpurun_out/bench_dist_cfg2.json 2> gpurun_out/bench_dist_cfg2.err; tail -c 1500 gpurun_out/bench_dist_cfg2.json; tail -3 gpurun_out/bench_dist_cfg2.err
timeout 900 python bench.py --config 3 --force-distributed --steps 3 --warmup 2 > gpurun_out/bench_dist_cfg3.json 2> gpurun_out/bench_dist_cfg3.err; tail -c 600 gpurun_out/bench_dist_cfg3.json; tail -3 gpurun_out/bench_dist_cfg3.err
