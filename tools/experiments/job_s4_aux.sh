set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python tools/emu_profile.py 16384 16384 4096 1 14 0 8192 0 > gpurun_out/s4_emu_prof.log 2>&1
timeout 900 $NCU --set full --clock-control none -k "regex:k_crt_split_cols|k_crt_split_rows|k_crt_accum|k_crt_col_scale|k_crt_row_scale" -c 5 -o gpurun_out/s4_aux_kernels -f python tools/emu_profile.py 16384 16384 4096 1 14 0 8192 0 > gpurun_out/s4_ncu_aux.log 2>&1; tail -1 gpurun_out/s4_ncu_aux.log
cat gpurun_out/s4_emu_prof.log
