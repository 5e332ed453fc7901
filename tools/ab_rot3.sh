#!/bin/bash
# A/B/C of the pair kernel's wave order (FN_GEMM2_TILE_ROT = 0 plain, 1 rotated, 2 matched table).
SH=${1:-"[(4096,4096,28672),(2048,4096,16384),(8192,8192,57344)]"}
for i in 1 2 3; do
  for r in 0 1 2; do
    echo "== FN_GEMM2_TILE_ROT=$r (pass $i)"
    FN_GEMM2_TILE_ROT=$r timeout 300 python tools/ab_prefill.py "$SH" 2>&1 | sed 's# dyt-prologue[^ ]*##g'
  done
done
