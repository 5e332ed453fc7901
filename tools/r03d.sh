#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r03e.log 2>&1 || { tail -30 gpurun_out/build_r03e.log; exit 1; }
for v in 10 11 12; do FN_FOLD_VARIANT=$v timeout 300 python tools/check_k1.py 2>&1 | tail -3; done
for rep in 1 2; do for v in 0 10 11 12; do FN_FOLD_VARIANT=$v timeout 120 python tools/ab_fold.py 2>&1; done; done | tee gpurun_out/ab_fold_r03e.txt
