python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02c.log 2>&1 || { tail -30 gpurun_out/build_r02c.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fold_mean_center_kernel" -s 2 -c 1 -o gpurun_out/prof_k2_r02e -f python tools/prof_folds.py > gpurun_out/ncu_k2_r02e.log 2>&1; echo "ncu_exit=$?"
