"""fold_mean_center 4096x4096 bf16 a few times (for per-kernel ncu timing)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
x, Vt, bp = SD.upstream(4, 16, n, n, "cuda", torch.bfloat16)
Vs = torch.empty_like(Vt)
ws = torch.zeros(fn.fold_mean_center_workspace_bytes(n, n) // 8 + 2, dtype=torch.float64, device="cuda")
for _ in range(4):
    fn.fold_mean_center(Vt, bp, out=Vs, workspace=ws)
torch.cuda.synchronize()
