"""Runs the folds a few times (for ncu per-kernel timing)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
dev = "cuda"
x, Vt, bp = SD.upstream(4, 16, 4096, 4096, dev, torch.bfloat16)
W, g, b, c = SD.layer(3, 28672, 4096, dev, torch.bfloat16, with_b=True, with_c=True)
a = SD.activations(3, 4096, 4096, dev, torch.bfloat16)
ws = torch.zeros(fn.linear_workspace_bytes(4096, 4096, 4096, "dyt", torch.bfloat16), dtype=torch.uint8, device=dev)
for _ in range(3):
    fn.fold_mean_center(Vt, bp)
    fn.fold_weights(W, g, b, c)
    fn.linear(a, W[:4096], None, mode="dyt", workspace=ws)
torch.cuda.synchronize()
