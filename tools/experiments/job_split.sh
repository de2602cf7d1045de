for v in 0 1; do echo "== HPS_SPLIT_FLOOR=$v"; HPS_SPLIT_FLOOR=$v python tools/bench_inverse.py 2>&1 | grep -E "inverse n=( 256| 512| 1024| 2048) batch=     1|512x512x512|256x256x256|1024x4096|512x2048"; done
for i in 1 2; do for v in 0 1; do echo "== HPS_SPLIT_FLOOR=$v cfg2"; HPS_SPLIT_FLOOR=$v python tools/stage_times.py 2 2>&1 | grep -E "device total|solve"; done; done
for v in 0 1; do echo "== HPS_SPLIT_FLOOR=$v cfg3"; HPS_SPLIT_FLOOR=$v python tools/stage_times.py 3 2>&1 | grep -E "device total|solve"; done
for v in 0 1; do echo "== HPS_SPLIT_FLOOR=$v cfg4"; HPS_SPLIT_FLOOR=$v python tools/stage_times.py 4 2>&1 | grep -E "device total|solve"; done
