python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02e.log 2>&1 || { tail -30 gpurun_out/build_r02e.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "stream_k" --timeout 60 -p no:cacheprovider 2>&1 | tail -5
for rep in 1 2; do for v in 0 1; do FN_GEMM2_SK=$v timeout 120 python tools/ab_prefill.py "[(2048,4096,4096),(2048,4096,16384),(4096,4096,28672)]" 2>&1 | sed "s/^/SK=$v /"; done; done
