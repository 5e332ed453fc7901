#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02q.log 2>&1 || { tail -30 gpurun_out/build_r02q.log; exit 1; }
python tools/host_overhead.py 2>&1 | tee gpurun_out/host_overhead_r02q.txt
bash tools/ab_local.sh 2>&1 | tee gpurun_out/ab_local_r02q.txt
