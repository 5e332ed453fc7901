"""Decode kernel with W* L2-resident (same 50 MB W* every call): exposes the compute rate
of the GEMV path, separately from HBM.  CUDA graph of 200 calls."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
K, N = 4096, 6144
w, g, _, _ = SD.layer(100, N, K, "cuda", torch.bfloat16)
W = fn.fold_weights(w, g)[0]
for M in (1, 16):
    a = SD.activations(7, M, K, "cuda", torch.bfloat16)
    z = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    for _ in range(10):
        fn.linear(a, W, None, out=z)
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st), torch.cuda.graph(gr, stream=st):
        for _ in range(200):
            fn.linear(a, W, None, out=z)
    gr.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); gr.replay(); e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) / 200 * 1e3
    print(f"L2-resident W* M={M}: {us:.2f} us/call  ({K * N * 2 / us / 1e3:.0f} GB/s)")
