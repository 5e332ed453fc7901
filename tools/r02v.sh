#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02v.log 2>&1 || { tail -30 gpurun_out/build_r02v.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_layernorm.py tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -3 | tee gpurun_out/pytest_r02v.log
for i in 1 2; do for l in 0 1; do FN_GEMM2_RMS_LOCAL=$l timeout 300 python tools/ab_ln.py; done; done 2>&1 | tee gpurun_out/ab_ln_r02v.txt
