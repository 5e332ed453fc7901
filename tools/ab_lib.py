"""A/B two source trees (each with its in-tree build), alternating runs on one box (same clocks):
    python tools/ab_lib.py TREE_A TREE_B      (e.g. `git archive HEAD | tar -x -C ab/A`, then build there)
config-3 prefill (rmsnorm, none) and config-2 decode (graph of 200 PDL-chained calls)."""
import os
import subprocess
import sys

CHILD = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
dev = "cuda"
def timed(f, steps=20, warm=5):
    for _ in range(warm): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / steps * 1e3
M, K, N = 4096, 4096, 28672
a = SD.activations(1, M, K, dev, torch.bfloat16)
W, g, _, _ = SD.layer(1, N, K, dev, torch.bfloat16)
Ws, cs = fn.fold_weights(W, g)
del W
z = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
r = timed(lambda: fn.linear(a, Ws, cs, out=z))
n = timed(lambda: fn.linear(a, Ws, cs, mode="none", out=z))
Wd = [fn.fold_weights(*SD.layer(100 + i, 6144, 4096, dev, torch.bfloat16)[:2])[0] for i in range(4)]
ad = SD.activations(7, 1, 4096, dev, torch.bfloat16)
zd = torch.empty(1, 6144, dtype=torch.bfloat16, device=dev)
st = torch.cuda.Stream()
gr = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    fn.linear(ad, Wd[0], None, out=zd); torch.cuda.synchronize()
    with torch.cuda.graph(gr, stream=st):
        for i in range(200): fn.linear(ad, Wd[i % 4], None, out=zd)
gr.replay(); torch.cuda.synchronize()
d = timed(lambda: gr.replay(), steps=3, warm=1) / 200
print(f"{sys.argv[1]}: prefill rms {2*M*K*N/r/1e6:.0f} none {2*M*K*N/n/1e6:.0f} TFLOP/s | decode M=1 {d:.2f} us", flush=True)
'''

if __name__ == "__main__":
    for rep in range(3):
        for tree in sys.argv[1:]:
            subprocess.run([sys.executable, "-c", CHILD, tree], cwd=tree, check=False)
