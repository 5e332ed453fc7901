"""Mode none vs rmsnorm on a K = 8192 shape, interleaved in one process (checks order / power effects)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
dev = "cuda"
def timed(f, steps=10, warm=3):
    for _ in range(warm): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / steps * 1e3
for (M, K, N) in [(8192, 8192, 28672), (4096, 8192, 28672), (8192, 4096, 28672)]:
    a = SD.activations(1, M, K, dev, torch.bfloat16)
    W, g, b, c = SD.layer(1, N, K, dev, torch.bfloat16, with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(W, g, b, c)
    del W
    z = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    out = []
    for mode in ("none", "rmsnorm", "none", "rmsnorm", "none"):
        us = timed(lambda: fn.linear(a, Ws, cs, mode=mode, path="gemm", out=z))
        out.append(f"{mode}={2*M*K*N/us/1e6:.0f}")
    print(f"M={M} K={K} N={N} TFLOP/s: " + " ".join(out), flush=True)
