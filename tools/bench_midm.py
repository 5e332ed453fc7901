"""Batched decode / short prefill shapes (M = 16 .. 256) at config 2's K = 4096, N = 6144: per call (CUDA graph
of back-to-back calls over 8 rotating W*), GB/s of the W* stream and the path the library picks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

HBM = float(os.environ.get("HBM_GBS", "6549"))
K, N, NB = 4096, 6144, 8
Wd = [fn.fold_weights(*SD.layer(100 + r, N, K, "cuda", torch.bfloat16)[:2])[0] for r in range(NB)]


def graph_us(f, reps=40):
    for i in range(3):
        f(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
        for i in range(reps):
            f(i)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for M in (16, 17, 24, 32, 48, 64, 96, 128, 192, 256):
    a = SD.activations(7, M, K, "cuda", torch.bfloat16)
    z = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    for path in ("auto", "gemm1", "gemm") if M > 16 else ("auto",):
        try:
            us = graph_us(lambda i: fn.linear(a, Wd[i % NB], None, out=z, path=path))
        except Exception as ex:  # noqa: BLE001
            print(f"M={M} path={path}: {ex}")
            continue
        byts = K * N * 2 + M * K * 2 + M * N * 2
        print(f"M={M:4d} path={path:6s}: {us:7.2f} us  {byts / us / 1e3:6.0f} GB/s ({byts / us / 1e3 / HBM:.2f} of HBM)"
              f"  {2 * M * K * N / us / 1e6:6.1f} TFLOP/s", flush=True)
