#!/bin/bash
# K1 variants A/B + copy ceilings at the fold sizes
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02j.log 2>&1 || { tail -30 gpurun_out/build_r02j.log; exit 1; }
for rep in 1 2; do for v in 0 10 11 12 13 14 15 9; do FN_FOLD_VARIANT=$v timeout 120 python tools/ab_fold.py 2>&1; done; done | tee gpurun_out/ab_fold_r02j.txt
timeout 300 python tools/bench_folds.py 2>&1 | tee gpurun_out/bench_folds_r02j.txt
