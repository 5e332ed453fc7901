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
HBM = 6544.0


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


def rotating(n, make):
    return [make(i) for i in range(n)]


for (n_out, d_in) in ((4096, 4096), (8192, 8192), (6144, 4096), (4096, 14336)):
    nbuf = max(2, -(-3 * 126 * 2 ** 20 // (2 * n_out * d_in * 2)))  # >= 3x L2 of V + V*
    Vts = rotating(nbuf, lambda i: SD.upstream(4 + i, 16, d_in, n_out, dev, torch.bfloat16)[1:])
    Vss = [torch.empty_like(v[0]) for v in Vts]
    ws = torch.zeros(fn.fold_mean_center_workspace_bytes(n_out, d_in) // 8 + 2, dtype=torch.float64, device=dev)
    it = [0]

    def f():
        i = it[0] % nbuf
        it[0] += 1
        fn.fold_mean_center(Vts[i][0], Vts[i][1], out=Vss[i], workspace=ws)
    us = graph_time(f, reps=4 * nbuf)
    byts = 2 * n_out * d_in * 2
    print(f"fold_mean_center {n_out}x{d_in} bf16 ({nbuf} rotating): {us:.1f} us  {byts / us / 1e3:.0f} GB/s  "
          f"({byts / us / 1e3 / HBM:.2f} of HBM)", flush=True)
    del Vts, Vss

for (N, K) in ((28672, 4096), (6144, 4096), (4096, 14336)):
    nbuf = max(1, -(-3 * 126 * 2 ** 20 // (2 * N * K * 2)))
    Ls = rotating(nbuf, lambda i: SD.layer(3 + i, N, K, dev, torch.bfloat16, with_b=True, with_c=True))
    Ws = [torch.empty_like(L[0]) for L in Ls]
    cs = torch.empty(N, device=dev)
    it = [0]

    def f():
        i = it[0] % nbuf
        it[0] += 1
        W, g, b, c = Ls[i]
        fn.fold_weights(W, g, b, c, out=Ws[i], c_out=cs)
    us = graph_time(f, reps=max(10, 4 * nbuf))
    byts = 2 * N * K * 2 + 4 * (2 * K + 2 * N)
    print(f"fold_weights {N}x{K} bf16 (g,b,c) ({nbuf} rotating): {us:.1f} us  {byts / us / 1e3:.0f} GB/s  "
          f"({byts / us / 1e3 / HBM:.2f} of HBM)", flush=True)
    del Ls, Ws

# ceilings at the same sizes: a plain device copy (torch copy_, read + write bytes) over rotating
# buffers, the same graph timing — what any two-stream (read + write) kernel of this size can reach
for nbytes in (2 * 4096 * 4096, 2 * 8192 * 8192, 2 * 28672 * 4096):
    nbuf = max(2, -(-3 * 126 * 2 ** 20 // (2 * nbytes)))
    srcs = [torch.empty(nbytes // 2, dtype=torch.bfloat16, device=dev).normal_() for _ in range(nbuf)]
    dsts = [torch.empty_like(s) for s in srcs]
    it = [0]

    def f():
        i = it[0] % nbuf
        it[0] += 1
        dsts[i].copy_(srcs[i])
    us = graph_time(f, reps=4 * nbuf)
    print(f"copy ceiling {nbytes / 1e6:.1f} MB -> {nbytes / 1e6:.1f} MB ({nbuf} rotating): {us:.1f} us  "
          f"{2 * nbytes / us / 1e3:.0f} GB/s  ({2 * nbytes / us / 1e3 / HBM:.2f} of HBM)", flush=True)
    del srcs, dsts
