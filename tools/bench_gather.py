"""Cost of the fused-gather epilogue (flashnorm_linear_gather) on one GPU: config-5 shard of
P = 8 (M = K = 8192, N_local = 7168) written to ndst LOCAL destinations (ndst x 117 MB of extra
HBM stores) vs the plain linear.  On a multi-GPU node ndst - 1 of these are NVLink peer stores."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

dev = "cuda"
M, K, Nl, P = 8192, 8192, 7168, 8
a = SD.activations(1, M, K, dev, torch.bfloat16)
W, g, _, _ = SD.layer(1, Nl, K, dev, torch.bfloat16)
Ws, cs = fn.fold_weights(W, g)
del W
z = torch.empty(M, Nl, dtype=torch.bfloat16, device=dev)
dsts = [torch.empty(M, Nl * P, dtype=torch.bfloat16, device=dev) for _ in range(P)]


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
    return s.elapsed_time(e) / steps


fl = 2.0 * M * K * Nl
t0 = timed(lambda: fn.linear(a, Ws, cs, out=z))
print(f"linear (z [M, N_local]): {t0 * 1e3:.0f} us  {fl / t0 / 1e9:.0f} TFLOP/s", flush=True)
for nd in (1, 2, 4, 8):
    t = timed(lambda: fn.linear_gather(a, Ws, dsts[:nd], 3 * Nl, c_star=cs))
    print(f"linear_gather ndst={nd} (+{nd * M * Nl * 2 / 1e6:.0f} MB stores): {t * 1e3:.0f} us  "
          f"{fl / t / 1e9:.0f} TFLOP/s  ({t / t0:.3f}x)", flush=True)
