python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02d.log 2>&1 || { tail -30 gpurun_out/build_r02d.log; exit 1; }
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "gemv or config2 or decode" --timeout 100 -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_rope.py tests/test_gpu_glu.py tests/test_gpu_layernorm.py -q -x --timeout 100 -p no:cacheprovider 2>&1 | tail -2
for n in 57344 75776; do for m in rmsnorm dyt; do FN_DECODE_VERBOSE=1 timeout 120 python tools/bench_decode.py $n $m 2>&1 | sort -u | grep "plan\|M=1 \|M=16"; done; done
