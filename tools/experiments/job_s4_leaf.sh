set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_spec.py -m gpu -x -q > gpurun_out/s4_leaf_tests.log 2>&1; tail -2 gpurun_out/s4_leaf_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
