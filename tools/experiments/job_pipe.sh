python -m pytest tests -m gpu -x -q -k "pipeline or capi or graph" > gpurun_out/pytest_pipe.log 2>&1; tail -3 gpurun_out/pytest_pipe.log
for s in 1 2 3 4 2 3; do echo "streams=$s"; HPS_PIPE_STREAMS=$s python tools/pipeline_probe.py 2 16 g 2>&1 | grep "jobs:" | head -1; done > gpurun_out/pipe_ab.txt 2>&1
for s in 2 3; do echo "streams=$s cfg3"; HPS_PIPE_STREAMS=$s python tools/pipeline_probe.py 3 8 g 2>&1 | grep "jobs:" | head -1; done >> gpurun_out/pipe_ab.txt 2>&1
for s in 2 3; do echo "streams=$s cfg4"; HPS_PIPE_STREAMS=$s python tools/pipeline_probe.py 4 4 g 2>&1 | grep "jobs:" | head -1; done >> gpurun_out/pipe_ab.txt 2>&1
