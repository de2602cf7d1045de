for i in 1 2; do for v in 128 64; do echo "== HPS_INV_BASE=$v cfg2"; HPS_INV_BASE=$v python tools/stage_times.py 2 2>&1 | grep -E "merge_d[0-5] |device total"; done; done
for v in 128 64; do echo "== HPS_INV_BASE=$v cfg3"; HPS_INV_BASE=$v python tools/stage_times.py 3 2>&1 | grep -E "device total"; done
python tools/bench_inverse.py > gpurun_out/bench_inverse.txt 2>&1; tail -20 gpurun_out/bench_inverse.txt
