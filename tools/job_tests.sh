# GPU tests + smoke (any round): logs under gpurun_out/
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
grep -E "diff .* gate" gpurun_out/pytest_gpu.log | head -40
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
