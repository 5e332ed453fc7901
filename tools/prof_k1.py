"""One config-3 fold_weights call (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

W, g, b, c = SD.layer(3, 28672, 4096, "cuda", torch.bfloat16, with_b=True, with_c=True)
Ws = torch.empty_like(W)
cs = torch.empty(28672, device="cuda")
for _ in range(3):
    fn.fold_weights(W, g, b, c, out=Ws, c_out=cs)
torch.cuda.synchronize()
