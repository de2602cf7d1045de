set -x
for cps in 1 2; do for per in 0 1; do
  echo "== CTAS_PER_SM=$cps PERSIST=$per"
  HPS_LEAF3_CTAS_PER_SM=$cps HPS_LEAF_L2PERSIST=$per python tools/stage_times.py 2 2>&1 | grep -E "leaf|device total"
done; done
for cps in 1 2; do for per in 0 1; do
  HPS_LEAF3_CTAS_PER_SM=$cps HPS_LEAF_L2PERSIST=$per timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum --clock-control none -k regex:k_leaf16v3 -c 1 --csv python tools/stage_times.py 2 > gpurun_out/ncu_leaf_${cps}_${per}.csv 2>/dev/null
  echo "ncu cps=$cps per=$per"; grep -E "dram__|gpu__time|lts__" gpurun_out/ncu_leaf_${cps}_${per}.csv | awk -F'","' '{print $(NF-2), $NF}'
done; done
