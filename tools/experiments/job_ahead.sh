# A/B of the look-ahead interface inverse (HPS_AHEAD_MIN_N3: 0 = off; HPS_GJ_RESERVE: SM reservation)
python -m pytest tests -m gpu -x -q -k "parity or pipeline or spec" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
echo "== off cfg2"; HPS_AHEAD_MIN_N3=0 python tools/stage_times.py 2 2>&1 | grep -E "merge_d[0-5] |device total"
echo "== ahead, reserve cfg2"; python tools/stage_times.py 2 2>&1 | grep -E "merge_d[0-5] |device total"
echo "== ahead, no reserve cfg2"; HPS_GJ_RESERVE=0 python tools/stage_times.py 2 2>&1 | grep -E "merge_d[0-5] |device total"
done
echo "== off cfg3"; HPS_AHEAD_MIN_N3=0 python tools/stage_times.py 3 2>&1 | grep -E "device total"
echo "== ahead cfg3"; python tools/stage_times.py 3 2>&1 | grep -E "device total"
echo "== ahead max 2048 cfg3"; HPS_AHEAD_MAX_N3=2048 python tools/stage_times.py 3 2>&1 | grep -E "device total"
echo "== off cfg4"; HPS_AHEAD_MIN_N3=0 python tools/stage_times.py 4 2>&1 | grep -E "device total"
echo "== ahead cfg4"; python tools/stage_times.py 4 2>&1 | grep -E "device total"
for s in 2; do echo "e2e cfg2 streams=$s"; python tools/pipeline_probe.py 2 16 g 2>&1 | grep "jobs:" | head -1; echo "e2e cfg2 off"; HPS_AHEAD_MIN_N3=0 python tools/pipeline_probe.py 2 16 g 2>&1 | grep "jobs:" | head -1; done
