#!/bin/bash
bash tools/gpu_round.sh r03u
REPS=20 timeout 900 python tools/stress.py 2>&1 | tail -3 | tee gpurun_out/stress_r03u.txt
timeout 200 python tools/bench_midm.py 2>&1 | tee gpurun_out/midm_r03u.txt
for i in 1 2; do timeout 300 python tools/ab_ln.py; done 2>&1 | tee gpurun_out/ab_ln_r03u.txt
