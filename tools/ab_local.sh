#!/bin/bash
# A/B of FN_GEMM2_RMS_LOCAL under the matched wave order, alternating processes.
SH="[(4096,4096,28672),(2048,4096,16384),(8192,8192,28672)]"
for i in 1 2 3; do
  for r in 0 1; do
    echo "== FN_GEMM2_RMS_LOCAL=$r (pass $i)"
    FN_GEMM2_RMS_LOCAL=$r timeout 300 python tools/ab_prefill.py "$SH" 2>&1 | sed -E 's# (dyt-prologue|dyt-prepass)[^ ]*##g; s# (rmsnorm|none)/gemm1=[0-9]*##g'
  done
done
