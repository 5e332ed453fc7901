python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02f.log 2>&1 || { tail -30 gpurun_out/build_r02f.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -p no:cacheprovider -k "stream_k or linear or gather" 2>&1 | tail -3
for rep in 1 2; do for v in "0 0" "0 1" "1 0" "1 1"; do set -- $v; FN_GEMM2_SK=$1 FN_GEMM2_STG=$2 timeout 120 python tools/ab_prefill.py "[(2048,4096,4096),(4096,4096,28672),(8192,8192,28672)]" 2>&1 | sed "s/^/SK=$1 STG=$2 /" | sed 's/ dyt-prologue.*//'; done; done
