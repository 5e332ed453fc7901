#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02m.log 2>&1 || { tail -30 gpurun_out/build_r02m.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "fold_mean_center or config4" 2>&1 | tail -5 | tee gpurun_out/pytest_r02m.log
timeout 300 python tools/bench_folds.py 2>&1 | tee gpurun_out/bench_folds_r02m.txt
FN_K2_VARIANT=3 timeout 300 python tools/bench_folds.py 2>&1 | grep mean_center | sed 's/^/3k: /' | tee -a gpurun_out/bench_folds_r02m.txt
