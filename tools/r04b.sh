#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r04b.log 2>&1 || { tail -30 gpurun_out/build_r04b.log; exit 1; }
for rep in 1 2 3; do for v in 0 1; do echo "== PDL_LATE=$v"; DECODE_MS=1,2,4,8,12,16 FN_DECODE_PDL_LATE=$v timeout 120 python tools/bench_decode.py 2>&1 | grep "M="; done; done 2>&1 | tee gpurun_out/pdl_late_r04b.txt
