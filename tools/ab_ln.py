"""A/B of the RMS / exact-LayerNorm pair kernel per call (graph of back-to-back calls, random data).

    FN_GEMM2_RMS_LOCAL=1 python tools/ab_ln.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402


def timed(f, steps=20):
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            for _ in range(steps):
                f()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps * 1e3


tag = os.environ.get("FN_GEMM2_RMS_LOCAL", "1")
for (M, K, N) in ((2048, 4096, 4096), (4096, 4096, 28672), (2048, 4096, 16384)):
    a = SD.activations(9, M, K, "cuda", torch.bfloat16)
    W, g, _, _ = SD.layer(9, N, K, "cuda", torch.bfloat16)
    Ws, cs = fn.fold_weights(W, g)
    u = fn.fold_colsum(Ws)
    z = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    us_ln = timed(lambda: fn.layernorm_linear(a, Ws, u, cs, eps=1e-5, out=z))
    us_rms = timed(lambda: fn.linear(a, Ws, cs, eps=1e-5, out=z))
    fl = 2.0 * M * K * N
    print(f"local={tag} M={M} K={K} N={N}: exact LN {us_ln:.1f} us ({fl / us_ln / 1e6:.0f} TFLOP/s)  "
          f"rms {us_rms:.1f} us ({fl / us_rms / 1e6:.0f} TFLOP/s)", flush=True)
