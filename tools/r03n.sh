#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r03n.log 2>&1 || { tail -30 gpurun_out/build_r03n.log; exit 1; }
timeout 60 ./tools/micro/k2p_trace 4096 | tail -9 | tee gpurun_out/k2p_trace_r03n.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "fold_mean_center" 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/bench_folds.py 2>&1 | grep "mean_center"; done | tee -a gpurun_out/k2p_trace_r03n.txt
