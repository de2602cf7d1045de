# A/B: K <= 32 GEMMs on the 2-stage / 4-CTA-per-SM config (HPS_SMALLK=1) vs the default config
for i in 1 2; do for v in 0 1; do echo "== HPS_SMALLK=$v cfg2"; HPS_SMALLK=$v python tools/stage_times.py 2 2>&1 | grep -E "merge_d(6|7|8|9|10|11) |device total"; done; done
for v in 0 1; do echo "== HPS_SMALLK=$v cfg4"; HPS_SMALLK=$v python tools/stage_times.py 4 2>&1 | grep -E "merge_d(11|12|13|14|15) |device total"; done
python -m pytest tests -m gpu -x -q -k "gemm or parity" 2>&1 | tail -2
