# Round 2, first GPU call: tests of the round-1 state, the new default bench line (config 5), the
# reference arm (sampled model) and its validation, the launch list and the depth-0 T GEMM capture.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; tail -c 600 gpurun_out/bench_cfg5.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_cfg5.json 2> gpurun_out/bench_ref_cfg5.err; tail -c 400 gpurun_out/bench_ref_cfg5.json
python bench.py --validate-reference-model > gpurun_out/ref_model_validation.json 2> gpurun_out/ref_model_validation.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench_cfg5.csv python tools/one_build.py 5 > gpurun_out/ncu_bench.log 2>&1
bash tools/ncu_top_gemm_cfg5.sh
echo done
