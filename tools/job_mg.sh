set -u
timeout 900 python -m pytest tests/test_gpu_multigpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --config 3 --force-distributed --steps 3 --warmup 2 2>/dev/null | tail -1 | cut -c1-300
