"""Device time of the folds (K1, K2) without host launch overhead: CUDA graph of back-to-back
calls with preallocated outputs/workspace, CUDA events on the capturing stream.

    python tools/bench_folds.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

dev = torch.device("cuda", 0)
HBM = 6553.3


def graph_time(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
        for _ in range(reps):
            f()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for (n_out, d_in) in ((4096, 4096), (8192, 8192), (6144, 4096)):
    x, Vt, bp = SD.upstream(4, 16, d_in, n_out, dev, torch.bfloat16)
    Vs = torch.empty_like(Vt)
    ws = torch.empty(fn.fold_mean_center_workspace_bytes(n_out, d_in) // 8 + 2, dtype=torch.float64, device=dev)
    us = graph_time(lambda: fn.fold_mean_center(Vt, bp, out=Vs, workspace=ws))
    byts = 2 * n_out * d_in * 2
    print(f"fold_mean_center {n_out}x{d_in} bf16: {us:.1f} us  {byts / us / 1e3:.0f} GB/s  "
          f"({byts / us / 1e3 / HBM:.2f} of HBM)", flush=True)

for (N, K) in ((28672, 4096), (6144, 4096)):
    W, g, b, c = SD.layer(3, N, K, dev, torch.bfloat16, with_b=True, with_c=True)
    Ws = torch.empty_like(W)
    cs = torch.empty(N, device=dev)
    us = graph_time(lambda: fn.fold_weights(W, g, b, c, out=Ws, c_out=cs), reps=10)
    byts = 2 * N * K * 2 + 4 * (2 * K + 2 * N)
    print(f"fold_weights {N}x{K} bf16 (g,b,c): {us:.1f} us  {byts / us / 1e3:.0f} GB/s  "
          f"({byts / us / 1e3 / HBM:.2f} of HBM)", flush=True)
