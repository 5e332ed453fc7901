"""RMS prefill TFLOP/s on the BASELINE shapes in one process (A/B knob comparisons run this in
alternating processes): config 3, config 4 (N = 4096), config-5 8-rank shard, config 5 on one GPU."""
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


out = []
for (M, K, N) in [(4096, 4096, 28672), (2048, 4096, 4096), (8192, 8192, 7168), (8192, 8192, 57344)]:
    a = SD.activations(1, M, K, dev, torch.bfloat16)
    W, g, _, _ = SD.layer(1, N, K, dev, torch.bfloat16)
    Ws, _ = fn.fold_weights(W, g)
    del W
    z = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    us = timed(lambda: fn.linear(a, Ws, None, out=z), steps=5 if N > 30000 and K > 4096 else 10)
    out.append(f"{M}x{K}x{N}={2 * M * K * N / us / 1e6:.0f}")
    del a, Ws, z
    torch.cuda.empty_cache()
print(os.environ.get("TAG", ""), " ".join(out), flush=True)
