# Round-1 measurement refresh (session 2): all five configs, the reference arm, the ncu launch list of
# the bench command and one full ncu capture of the leaf kernel.
set -u
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for c in 1 3 4; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; done
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_leaf16v3 -c 1 -o gpurun_out/prof_leaf16v3_r01c python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_leaf_full.log 2>&1
echo done
