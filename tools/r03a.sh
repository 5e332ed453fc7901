#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r03a.log 2>&1 || { tail -30 gpurun_out/build_r03a.log; exit 1; }
REPS=20 timeout 900 python tools/stress.py 2>&1 | tail -8 | tee gpurun_out/stress_r03a.txt
SH="[(4096,4096,28672),(8192,8192,57344),(2048,4096,16384)]"
for i in 1 2; do for sk in 0 2; do echo "== SK=$sk pass $i"; FN_GEMM2_SK=$sk timeout 300 python tools/ab_prefill.py "$SH" 2>&1 | sed -E 's# (dyt-prologue|dyt-prepass)[^ ]*##g; s# (rmsnorm|none)/gemm1=[0-9]*##g'; done; done | tee gpurun_out/ab_sk_r03a.txt
