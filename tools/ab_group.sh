#!/bin/bash
# A/B of balanced tile groups (FN_GEMM2_GROUP_BAL) on the config-5 shapes, alternating processes.
SH="[(8192,8192,57344),(8192,8192,28672),(8192,8192,14336),(8192,8192,7168)]"
for i in 1 2 3; do
  for r in 0 1; do
    echo "== FN_GEMM2_GROUP_BAL=$r (pass $i)"
    FN_GEMM2_GROUP_BAL=$r timeout 300 python tools/ab_prefill.py "$SH" 2>&1 | sed -E 's# (dyt-prologue|dyt-prepass|none)[^ ]*##g; s# rmsnorm/gemm1=[0-9]*##'
  done
done
