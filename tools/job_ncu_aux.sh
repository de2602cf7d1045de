set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none -k "regex:k_crt_split_cols|k_crt_split_rows|k_crt_accum|k_crt_col_scale" -c 4 -o gpurun_out/aux_kernels -f python tools/emu_profile.py 4096 4096 1024 64 14 0 8192 0 > gpurun_out/ncu_aux.log 2>&1; tail -1 gpurun_out/ncu_aux.log
