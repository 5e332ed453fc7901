python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02d.log 2>&1 || { tail -30 gpurun_out/build_r02d.log; exit 1; }
for pf in 12 16 23; do echo "L2PF=$pf"; FN_DECODE_L2PF=$pf timeout 120 python tools/bench_decode.py 6144 dyt 2>&1 | sort -u | grep "M=1 \|M=16"; done
