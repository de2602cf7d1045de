# A/B of two library builds on the same box: per-depth merge times and device totals (cfg2, cfg4)
for i in 1 2; do
  for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do
    echo "== $lib"; HPS_LIB=$PWD/$lib python tools/stage_times.py 2 2>&1 | grep -E "merge_d(0|2|5|8|10|11) |device total"
  done
done
for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do
  echo "== $lib cfg4"; HPS_LIB=$PWD/$lib python tools/stage_times.py 4 2>&1 | grep -E "device total"
done
