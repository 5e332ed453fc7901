#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02p.log 2>&1 || { tail -30 gpurun_out/build_r02p.log; exit 1; }
for o in 1 0; do echo "ROWS $o"; FN_K2P_ROWS=$o ./tools/micro/k2p_trace 4096 | tail -9; done 2>&1 | tee gpurun_out/k2p_trace_r02p.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "fold_mean_center or config4" 2>&1 | tail -3 | tee gpurun_out/pytest_r02p.log
for o in 1 0; do FN_K2P_ROWS=$o timeout 300 python tools/bench_folds.py 2>&1 | grep "mean_center" | sed "s/^/ROWS $o: /"; done | tee -a gpurun_out/k2p_trace_r02p.txt
