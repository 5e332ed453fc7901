#!/bin/bash
# One GPU session: tests, bench, ncu launch list and full captures (outputs in gpurun_out/).
# usage: tools/gpu_round.sh [tag]
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
echo "== pytest"; timeout 1200 python -u -m pytest tests -m gpu -x -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest_exit=$?" | tee -a gpurun_out/pytest_$TAG.log; tail -3 gpurun_out/pytest_$TAG.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke_exit=$?" | tee -a gpurun_out/smoke_$TAG.log
echo "== bench"; timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench_exit=$?"; cat gpurun_out/bench_$TAG.json
echo "== configs"; timeout 900 python tools/bench_configs.py > gpurun_out/configs_$TAG.txt 2>&1; echo "configs_exit=$?"
echo "== ncu launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary-iters 5 > /dev/null 2>&1; echo "ncu_launch_exit=$?"
echo "== ncu full gemm"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:flashnorm_gemm2?_kernel -s 3 -c 1 -o gpurun_out/prof_gemm_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --secondary-iters 5 > gpurun_out/ncu_gemm_$TAG.log 2>&1; echo "ncu_gemm_exit=$?"
echo "== ncu full gemv"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:flashnorm_gemv_tc_kernel -s 8 -c 1 -o gpurun_out/prof_gemv_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --secondary-iters 5 > gpurun_out/ncu_gemv_$TAG.log 2>&1; echo "ncu_gemv_exit=$?"
echo "== ncu full folds/dyt"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fold_weights_kernel|fold_mean_center_persist|k2_tiles_kernel|colsum_reduce_kernel|dyt_prepass" -c 6 -o gpurun_out/prof_aux_$TAG -f python tools/prof_folds.py > gpurun_out/ncu_aux_$TAG.log 2>&1; echo "ncu_aux_exit=$?"
ls -la gpurun_out
