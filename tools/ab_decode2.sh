#!/bin/bash
# A/B the decode ring depth (2 CTAs/SM when <= 5 stages) x K split cap x LSU prefetch (config 2).
for cfg in "0 8 1" "5 8 1" "5 8 0" "4 8 1" "4 8 0" "5 2 1" "5 2 0" "3 8 0" "0 8 1"; do
  set -- $cfg
  echo "== stages=$1 smax=$2 lsupf=$3"
  FN_DECODE_STAGES=$1 FN_DECODE_SMAX=$2 FN_DECODE_LSUPF=$3 FN_DECODE_VERBOSE=1 timeout 120 python tools/bench_decode.py 2>&1 | grep -E "decode|rror|plan"
done
