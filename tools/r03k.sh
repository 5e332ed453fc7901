#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r03k.log 2>&1 || { tail -30 gpurun_out/build_r03k.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_glu.py tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -3 | tee gpurun_out/pytest_r03k.log
timeout 300 python tools/ab_down.py 2>&1 | tee gpurun_out/ab_down_r03k.txt
