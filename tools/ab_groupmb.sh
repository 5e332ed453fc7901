#!/bin/bash
# A/B of the tile-group A budget (FN_GEMM2_GROUP_MB) on config 5 and config 3, alternating processes.
SH="[(8192,8192,57344),(8192,8192,28672),(8192,8192,7168),(4096,4096,28672)]"
for i in 1 2; do
  for r in 24 40 64; do
    echo "== FN_GEMM2_GROUP_MB=$r (pass $i)"
    FN_GEMM2_GROUP_MB=$r timeout 300 python tools/ab_prefill.py "$SH" 2>&1 | sed -E 's# (dyt-prologue|dyt-prepass|none)[^ ]*##g; s# rmsnorm/gemm1=[0-9]*##'
  done
done
