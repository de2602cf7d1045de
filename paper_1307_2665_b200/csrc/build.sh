#!/usr/bin/env bash
# Build libhps_b200.so in-tree for sm_100a (the .so travels to the GPU box with the repo).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
out="${HPS_OUT:-${here}/../libhps_b200.so}"
NVCC="${NVCC:-nvcc}"
FLAGS=(-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
       -I"${here}" -I"${here}/../../include" --expt-relaxed-constexpr ${HPS_NVCC_EXTRA:-})
objs=()
pids=()
mkdir -p "${HPS_OBJ:-${here}/../build_obj}"
for f in capi gemm emu i8gemm merge lu solve leaf leaf3 group post tree; do
  o="${HPS_OBJ:-${here}/../build_obj}/${f}.o"
  # tree.cu is host code that must reproduce numpy's fp64 results bit for bit: no FMA contraction
  extra=()
  [[ "$f" == tree ]] && extra=(-Xcompiler -ffp-contract=off)
  if [[ ! -f "$o" || "${here}/${f}.cu" -nt "$o" || "${here}/common.cuh" -nt "$o" || "${here}/gemm.cuh" -nt "$o" || "${here}/leaf.cuh" -nt "$o" || "${here}/ctx.cuh" -nt "$o" || "${here}/lu.cuh" -nt "$o" || "${here}/../../include/hps_b200.h" -nt "$o" ]]; then
    rm -f "$o"
    "$NVCC" "${FLAGS[@]}" "${extra[@]}" -c "${here}/${f}.cu" -o "$o" &
    pids+=($!)
  fi
  objs+=("$o")
done
for pid in "${pids[@]}"; do
  wait "$pid" || { echo "build.sh: compile failed" >&2; exit 1; }
done
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "${objs[@]}" -lcudart_static -L/usr/local/cuda/lib64 -lcublasLt -Xlinker -rpath -Xlinker /usr/local/cuda/lib64 -lrt -ldl -lpthread
echo "built $out"
