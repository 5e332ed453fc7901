#!/bin/bash
# Quick GPU session: pytest -m gpu, smoke, bench (outputs in gpurun_out/).  usage: tools/gpu_quick.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1
echo "== pytest"; timeout 900 python -u -m pytest tests -m gpu -x -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest_exit=$?" | tee -a gpurun_out/pytest_$TAG.log; tail -5 gpurun_out/pytest_$TAG.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke_exit=$?" | tee -a gpurun_out/smoke_$TAG.log
echo "== bench"; timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench_exit=$?"; cat gpurun_out/bench_$TAG.json; tail -5 gpurun_out/bench_$TAG.err
