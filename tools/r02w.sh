#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02w.log 2>&1 || { tail -30 gpurun_out/build_r02w.log; exit 1; }
for rep in 1 2; do
for v in "" "FN_DECODE_L2PF=16" "FN_DECODE_L2PF=24" "FN_DECODE_L2PF=40" "FN_DECODE_PF2=1" "FN_DECODE_PF2=1 FN_DECODE_L2PF=0"; do
  echo "== $v"; env $v timeout 120 python tools/bench_decode.py 2>&1 | grep -E "M=(1|16) "
done; done 2>&1 | tee gpurun_out/decode_knobs_r02w.txt
