#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r03t.log 2>&1 || { tail -30 gpurun_out/build_r03t.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "batched_decode" 2>&1 | tail -15
timeout 200 python tools/bench_midm.py 2>&1 | tee gpurun_out/midm_r03t.txt
