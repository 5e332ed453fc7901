"""The FFN down projection 4096 x 14336 -> 4096 (x s) per call: linear_scaled with the default
workspace (stream-K tail at K >= 8192) vs workspace=None (whole tiles), alternating, CUDA graphs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402


def timed(f, steps=10):
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


M, F, K = 4096, 14336, 4096
h = SD.activations(5, M, F, "cuda", torch.bfloat16)
Wd, _, _, _ = SD.layer(6, K, F, "cuda", torch.bfloat16)
s = torch.rand(M, device="cuda") + 0.5
z = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
ws = torch.zeros(fn.linear_workspace_bytes(M, F, K, "none", torch.bfloat16), dtype=torch.uint8, device="cuda")
fl = 2.0 * M * F * K
for rep in range(3):
    for tag, w in (("stream-K (default)", ws), ("whole tiles", None)):
        us = timed(lambda: fn.linear_scaled(h, Wd, s, out=z, workspace=w))
        print(f"down {tag}: {us:.1f} us {fl / us / 1e6:.0f} TFLOP/s", flush=True)
