#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02x.log 2>&1 || { tail -30 gpurun_out/build_r02x.log; exit 1; }
for v in 0 1 3 4 5 6 7 8; do FN_FOLD_VARIANT=$v timeout 120 python tools/ab_fold.py 2>&1; done | tee gpurun_out/ab_fold_r02x.txt
