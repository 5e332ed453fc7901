#!/bin/bash
# A/B of the pair kernel's rotated wave order (FN_GEMM2_TILE_ROT), alternating processes.
SH="[(4096,4096,28672),(2048,4096,16384),(2048,4096,4096),(8192,8192,28672),(8192,8192,7168)]"
for i in 1 2; do
  for r in 0 1; do
    echo "== FN_GEMM2_TILE_ROT=$r (pass $i)"
    FN_GEMM2_TILE_ROT=$r timeout 300 python tools/ab_prefill.py "$SH" 2>&1 | sed 's# dyt-prologue[^ ]*##g'
  done
done
