#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r03h.log 2>&1 || { tail -30 gpurun_out/build_r03h.log; exit 1; }
for rep in 1 2; do
for v in "" "FN_DECODE_L2PF=15" "FN_DECODE_L2PF=18" "FN_DECODE_L2PF=8" "FN_DECODE_TOKRES=0"; do
  echo "== dyt $v"; env $v FN_DECODE_VERBOSE=1 timeout 120 python tools/bench_decode.py 6144 dyt 2>&1 | grep -E "plan|M=(1|16) "
done; done 2>&1 | tee gpurun_out/decode_dyt_r03h.txt
