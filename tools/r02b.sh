python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02b.log 2>&1 || { tail -30 gpurun_out/build_r02b.log; exit 1; }
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "fold_mean or config4" --timeout 100 -p no:cacheprovider 2>&1 | tail -3
for v in 0 1; do echo "K2 variant $v"; FN_K2_VARIANT=$v timeout 200 python tools/bench_folds.py 2>&1 | grep mean_center; done
