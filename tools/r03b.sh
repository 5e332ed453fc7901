#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r03b.log 2>&1 || { tail -30 gpurun_out/build_r03b.log; exit 1; }
SH="[(4096,4096,28672),(4096,4096,14336)]"
for i in 1 2 3; do for sk in 0 2; do echo "== SK=$sk MAXW=64 pass $i"; FN_GEMM2_SK_MAXW=64 FN_GEMM2_SK=$sk timeout 300 python tools/ab_prefill.py "$SH" 2>&1 | sed -E 's# (dyt-prologue|dyt-prepass)[^ ]*##g; s# (rmsnorm|none)/gemm1=[0-9]*##g'; done; done | tee gpurun_out/ab_sk_r03b.txt
FN_GEMM2_SK_MAXW=64 FN_GEMM2_SK=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "config3 or stream_k or repeated" 2>&1 | tail -3
