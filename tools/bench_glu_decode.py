"""GLU FFN gate||up at decode / batched-decode sizes (K = 4096, F = 14336 -> Wgu 28672 rows): per call
(CUDA graph over rotating weights >= 3x L2), GB/s of the weight stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

HBM = float(os.environ.get("HBM_GBS", "6549"))
K, F, NB = 4096, 14336, 2
W = []
for r in range(NB):
    Wg = SD.layer(300 + r, F, K, "cuda", torch.bfloat16)[0]
    Wu = SD.layer(400 + r, F, K, "cuda", torch.bfloat16)[0]
    W.append(fn.fold_glu_weights(Wg, Wu, None))
    del Wg, Wu


def graph_us(f, reps=20):
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


for M in (1, 16, 32, 64, 128):
    a = SD.activations(7, M, K, "cuda", torch.bfloat16)
    h = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    s = torch.empty(M, dtype=torch.float32, device="cuda")
    us = graph_us(lambda i: fn.glu_linear(a, W[i % NB], eps=1e-5, act="silu", out=h, s_out=s))
    byts = 2 * F * K * 2
    print(f"glu gate||up M={M:3d}: {us:7.1f} us  {byts / us / 1e3:6.0f} GB/s ({byts / us / 1e3 / HBM:.2f} of HBM)", flush=True)
