#!/bin/bash
# A/B of FN_GEMM2_TILE_ROT on the config-5 shapes (multi-group tile order), alternating processes.
SH="[(8192,8192,57344),(8192,8192,28672),(4096,4096,28672)]"
for i in 1 2 3; do
  for r in 0 1; do
    echo "== FN_GEMM2_TILE_ROT=$r (pass $i)"
    FN_GEMM2_TILE_ROT=$r timeout 300 python tools/ab_prefill.py "$SH" 2>&1 | sed 's# dyt-prologue[^ ]*##g'
  done
done
