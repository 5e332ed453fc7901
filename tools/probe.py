"""Ad-hoc GPU probe: run one linear() configuration and report error vs the oracle.
usage: python tools/probe.py M K N mode path"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_09577_b200 as fn
from oracle import flashnorm_oracle as O
from synth import gen_activations, gen_layer
M, K, N = map(int, sys.argv[1:4]); mode = sys.argv[4]; path = sys.argv[5]
a = gen_activations(0, M, K, "normal", "bf16")
Wt, g, b, c = gen_layer(0, N, K, "bf16", with_b=True, with_c=True)
T = lambda x, bf=True: None if x is None else (torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16 if bf else torch.float32).cuda())
Ws, cs = fn.fold_weights(T(Wt), T(g, False), T(b, False), T(c, False))
torch.cuda.synchronize()
t0 = time.time()
z = fn.linear(T(a), Ws, cs, eps=1e-5, mode=mode, path=path)
torch.cuda.synchronize()
dt = time.time() - t0
rows = np.unique(np.r_[0, M - 1, np.arange(0, M, max(1, M // 16))])
ref = O.norm_linear(a[rows], Wt.T, g, b, c, 1e-5, mode)
print(f"probe M={M} K={K} N={N} {mode} {path}: err={O.rowwise_rel_err(z.float().cpu().numpy()[rows], ref):.3e} t={dt*1e3:.2f}ms", flush=True)
