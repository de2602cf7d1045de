set -u
timeout 900 python tools/pipeline_probe.py 5 4 graphs 2>&1 | grep -v -i warn | head -40
