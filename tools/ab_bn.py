"""Pair-kernel tile width A/B (FN_GEMM2_BN=256 vs the heuristic) on the BASELINE prefill shapes and
the column shards bench.py / config 5 produce (rmsnorm mode, TFLOP/s, one process per setting)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

dev = "cuda"


def timed(f, steps=10, warm=3):
    for _ in range(warm):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps * 1e3


shapes = [(4096, 4096, 28672), (4096, 4096, 14336), (4096, 4096, 7168), (4096, 4096, 3584), (2048, 4096, 4096), (2048, 4096, 16384),
          (8192, 8192, 14336), (8192, 8192, 7168)]
out = []
for (M, K, N) in shapes:
    a = SD.activations(1, M, K, dev, torch.bfloat16)
    W, g, _, _ = SD.layer(1, N, K, dev, torch.bfloat16)
    Ws, cs = fn.fold_weights(W, g)
    del W
    z = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    us = timed(lambda: fn.linear(a, Ws, cs, out=z))
    out.append(f"{M}x{K}x{N}: {2 * M * K * N / us / 1e6:.0f}")
    del a, Ws, z
print(f"BN={os.environ.get('FN_GEMM2_BN', 'auto')}: " + " | ".join(out), flush=True)
