"""Heavier determinism stress for the pair kernel's side group (RMS and exact LayerNorm, the formally
ordered own-barrier reads): REPS launches per shape must be bit-identical."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

reps = int(os.environ.get("REPS", "100"))
bad = 0
for (M, K, N) in [(2048, 4096, 4096), (4096, 4096, 28672), (9000, 256, 4096), (1000, 1000, 2048)]:
    a = SD.activations(5, M, K, "cuda", torch.bfloat16)
    W, g, b, c = SD.layer(5, N, K, "cuda", torch.bfloat16, with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(W, g, b, c)
    u = fn.fold_colsum(Ws)
    for tag, f in (("rmsnorm", lambda: fn.linear(a, Ws, cs, eps=1e-5)),
                   ("layernorm_linear", lambda: fn.layernorm_linear(a, Ws, u, cs, eps=1e-5))):
        z0 = f()
        nd = sum(int(not torch.equal(f(), z0)) for _ in range(reps))
        bad += nd > 0
        print(f"{'OK ' if nd == 0 else 'BAD'} M={M} K={K} N={N} {tag}: {nd}/{reps} launches differ", flush=True)
print("STRESS_LN", "PASS" if bad == 0 else f"FAIL ({bad})")
