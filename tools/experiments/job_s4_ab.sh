set -u
mkdir -p gpurun_out
run() { python bench.py --config 5 --no-cpu-baseline "$@" > gpurun_out/s4_ab.json 2> gpurun_out/s4_ab.err; python -c "
import json,sys; d=json.loads(open('gpurun_out/s4_ab.json').read().strip().splitlines()[-1]); print(sys.argv[1:], d['ms_per_step'], d['stages']['build_ms'], d['stages']['solve_ms'], d['clocks']['sm_mhz'])" "$@"; }
run --emu-min-k 256
run --emu-solve 1
run
