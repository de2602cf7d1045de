# A/B of two library builds on the same box: stage times of cfg2 and cfg4 (HPS_LIB selects the .so)
for i in 1 2; do
  for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do
    echo "== $lib"; HPS_LIB=$PWD/$lib python tools/stage_times.py 2 2>&1 | grep -E "leaf|device total"
  done
done
for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do
  echo "== $lib cfg4"; HPS_LIB=$PWD/$lib python tools/stage_times.py 4 2>&1 | grep -E "leaf |device total"
done
