python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02e.log 2>&1 || { tail -30 gpurun_out/build_r02e.log; exit 1; }
for rep in 1 2 3; do for v in 0 1; do TAG="local=$v" FN_GEMM2_RMS_LOCAL=$v timeout 120 python tools/ab_rms.py; done; done
FN_GEMM2_RMS_LOCAL=1 timeout 600 compute-sanitizer --tool racecheck --racecheck-report analysis python tools/sanitize.py "linear rmsnorm gemm" > gpurun_out/racecheck_local_r02e.log 2>&1; echo racecheck_exit=$?; grep -i "hazard\|ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/racecheck_local_r02e.log | tail -5
