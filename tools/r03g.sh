#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r03g.log 2>&1 || { tail -30 gpurun_out/build_r03g.log; exit 1; }
SH="[(4096,14336,4096),(2048,4096,4096),(8192,28672,8192)]"
for i in 1 2 3; do for sk in 0 2; do echo "== SK=$sk pass $i"; FN_GEMM2_SK=$sk timeout 300 python tools/ab_prefill.py "$SH" 2>&1 | sed -E 's# (dyt-prologue|dyt-prepass)[^ ]*##g; s# (rmsnorm|none)/gemm1=[0-9]*##g'; done; done | tee gpurun_out/ab_sk_r03g.txt
