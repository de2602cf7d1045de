for i in 1 2 3; do for lib in tools/libhps_b200_old.so tools/libhps_b200_cg.so; do echo "== $lib cfg2"; HPS_LIB=$PWD/$lib python tools/stage_times.py 2 2>&1 | grep -E "leaf "; done; done
for lib in tools/libhps_b200_old.so tools/libhps_b200_cg.so; do echo "== $lib cfg4"; HPS_LIB=$PWD/$lib python tools/stage_times.py 4 2>&1 | grep -E "leaf "; done
