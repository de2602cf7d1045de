for i in 1 2; do for v in 1 2 3 4; do echo "== HPS_SPLIT_DIV=$v cfg2"; HPS_SPLIT_DIV=$v python tools/stage_times.py 2 2>&1 | grep -E "device total|solve"; done; done
for v in 2 4; do echo "== HPS_SPLIT_DIV=$v cfg3"; HPS_SPLIT_DIV=$v python tools/stage_times.py 3 2>&1 | grep -E "device total"; done
for v in 1 2 4; do echo "== HPS_SPLIT_DIV=$v inv"; HPS_SPLIT_DIV=$v python tools/bench_inverse.py 2>&1 | grep -E "inverse n=( 512| 1024) batch=     1"; done
