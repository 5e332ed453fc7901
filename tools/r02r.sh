#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2407_09577_b200 import build; build.build()" > gpurun_out/build_r02r.log 2>&1 || { tail -30 gpurun_out/build_r02r.log; exit 1; }
python tools/host_overhead.py 2>&1 | tee gpurun_out/host_overhead_r02r.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02r.json 2> gpurun_out/bench_r02r.err; echo "bench_exit=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_r02r.json'))
print('value',d['value'],'frac',d['roofline']['frac'])
print('decode', {k:(round(v['us'],2),round(v['frac_hbm'],3),round(v['eager_us'],2),round(v['eager_frac_hbm'],3)) for k,v in d['decode'].items() if k.startswith('M')})
print('fold', d['fold'])
"
