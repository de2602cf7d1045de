# A/B of two library builds on the same box: inverse micro-benchmark + cfg2/cfg3 device totals
for i in 1 2; do
  for lib in tools/libhps_b200_old.so paper_1307_2665_b200/libhps_b200.so; do
    echo "== $lib"
    HPS_LIB=$PWD/$lib python tools/bench_inverse.py inv 2>&1 | grep -E "n=  128 batch=     1|n= 1024"
    HPS_LIB=$PWD/$lib python tools/stage_times.py 2 | grep "device total"
  done
done
