"""One prefill configuration for ncu: python tools/prof_one.py M K N mode [path]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
M, K, N = map(int, sys.argv[1:4]); mode = sys.argv[4]; path = sys.argv[5] if len(sys.argv) > 5 else "gemm"
a = SD.activations(1, M, K, "cuda", torch.bfloat16)
W, g, b, c = SD.layer(1, N, K, "cuda", torch.bfloat16, with_b=True, with_c=True)
Ws, cs = fn.fold_weights(W, g, b, c)
z = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(4):
    fn.linear(a, Ws, cs, mode=mode, path=path, out=z)
torch.cuda.synchronize()
