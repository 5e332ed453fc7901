#!/bin/bash
# A/B the decode kernel knobs (config 2): LSU prefetch (1 own, 2 partner, +4 evict_normal hint).
for cfg in "0 1" "0 5" "0 6" "0 7" "0 0" "0 1"; do
  set -- $cfg
  echo "== l2pf=$1 lsupf=$2"
  FN_DECODE_L2PF=$1 FN_DECODE_LSUPF=$2 python tools/bench_decode.py 2>&1 | grep decode
done
