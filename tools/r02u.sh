#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02u.log 2>&1 || { tail -30 gpurun_out/build_r02u.log; exit 1; }
for v in "" "FN_DECODE_TMAX=8" "FN_DECODE_SMAX=3 FN_DECODE_GLOBAL=1" "FN_DECODE_SMAX=2" "FN_DECODE_SMAX=4"; do
  echo "== $v"; env $v FN_DECODE_VERBOSE=1 timeout 120 python tools/bench_decode.py 2>&1 | grep -v "^$" | head -6
done 2>&1 | tee gpurun_out/decode_plans_r02u.txt
