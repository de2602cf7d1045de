HPS_LEAF_CHUNKS=4 HPS_PIPE_PRIO=1 python -m pytest tests -m gpu -x -q -k "pipeline or graph or parity" > gpurun_out/pytest_prio.log 2>&1; tail -2 gpurun_out/pytest_prio.log
for i in 1 2; do
for c in 1 4 8; do for pr in 0 1; do echo "chunks=$c prio=$pr"; HPS_LEAF_CHUNKS=$c HPS_PIPE_PRIO=$pr python tools/pipeline_probe.py 2 16 g 2>&1 | grep "jobs:" | head -1; done; done
done
for c in 1 4; do echo "device leaf chunks=$c"; HPS_LEAF_CHUNKS=$c python tools/stage_times.py 2 2>&1 | grep -E "leaf|device total"; done
for c in 1 4; do for pr in 0 1; do echo "cfg3 chunks=$c prio=$pr"; HPS_LEAF_CHUNKS=$c HPS_PIPE_PRIO=$pr python tools/pipeline_probe.py 3 8 g 2>&1 | grep "jobs:" | head -1; done; done
