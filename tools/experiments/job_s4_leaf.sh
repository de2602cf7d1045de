set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s4_leaf_tests.log 2>&1; tail -2 gpurun_out/s4_leaf_tests.log
for c in 2 2 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/s4_ab.json 2> gpurun_out/s4_ab.err; python -c "
import json,sys; d=json.loads(open('gpurun_out/s4_ab.json').read().strip().splitlines()[-1]); st=d['stages']; print($c, round(d['ms_per_step'],3), round(st['build_ms'],3), {k: round(v,3) for k,v in st.items() if 'leaf' in k and isinstance(v,(int,float))}, round(d['roofline']['achieved'],2))"; done
