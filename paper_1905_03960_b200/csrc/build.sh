#!/usr/bin/env bash
# Builds libp3.so (sm_100a) in-tree. Invoked by __graft_entry__.build().
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="${HERE}/../libp3.so"
NVCC="${NVCC:-/usr/local/cuda/bin/nvcc}"
FLAGS=(-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3
       -cudart static -shared -ldl -I"${HERE}/../../include" -Xptxas -v)
SRCS=("${HERE}/p3_host.cpp" "${HERE}/p3_sim.cpp" "${HERE}/p3_kernels.cu" "${HERE}/p3_ctx.cu" "${HERE}/p3_wire.cu")
# the checked build (protocol invariants compiled in, tests/test_gpu_checked.py) alongside
"${NVCC}" "${FLAGS[@]}" -DP3_CHECKS -o "${HERE}/../libp3_checked.so.tmp" "${SRCS[@]}" 2> "${HERE}/../ptxas_checked.log" &
CHECKED=$!
"${NVCC}" "${FLAGS[@]}" -o "${OUT}.tmp" "${SRCS[@]}" 2> "${HERE}/../ptxas.log" || {
  cat "${HERE}/../ptxas.log" >&2; exit 1; }
wait "${CHECKED}" || { cat "${HERE}/../ptxas_checked.log" >&2; exit 1; }
mv "${OUT}.tmp" "${OUT}"
mv "${HERE}/../libp3_checked.so.tmp" "${HERE}/../libp3_checked.so"
echo "built ${OUT} (+ libp3_checked.so)"
