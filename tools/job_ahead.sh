set -u
for c in 2 3; do
for cfg in "128 3.2e6" "0 0" "128 1.6e6" "128 1e7" "128 1e9" "256 3.2e6"; do
  set -- $cfg
  HPS_AHEAD_MIN_N3=$1 HPS_AHEAD_WORK=$2 timeout 600 python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print($c, '$1', '$2', round(d['ms_per_step'],3), round(d['stages']['build_ms'],3))"
done; done
for cfg in "128 3.2e6" "128 1e9"; do
  set -- $cfg
  HPS_AHEAD_MIN_N3=$1 HPS_AHEAD_WORK=$2 timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(4, '$1', '$2', round(d['ms_per_step'],3), round(d['stages']['build_ms'],3))"
done
