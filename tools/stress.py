"""Determinism/parity stress for the tcgen05 GEMM: repeated launches must be bit-identical."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
dev = "cuda"
bad = 0
for (M, K, N) in [(4096, 512, 28672), (256, 512, 28672), (4096, 1024, 28672), (4096, 4096, 28672), (2048, 64, 8192), (1000, 320, 4104)]:
    a = SD.activations(0, M, K, dev, torch.bfloat16)
    Wt, g, b, c = SD.layer(0, N, K, dev, torch.bfloat16, with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(Wt, g, b, c)
    af = a.float()
    for mode in ("rmsnorm", "dyt", "none"):
        z0 = fn.linear(a, Ws, cs, eps=1e-5, mode=mode, path="gemm")
        if mode == "rmsnorm":
            ref = (af @ Ws.float().T) * torch.rsqrt((af * af).mean(1, keepdim=True) + 1e-5) + cs
        elif mode == "none":
            ref = af @ Ws.float().T + cs
        else:
            ref = None
        nd = 0
        for rep in range(int(os.environ.get("REPS", "10"))):
            z = fn.linear(a, Ws, cs, eps=1e-5, mode=mode, path="gemm")
            nd += int(not torch.equal(z, z0))
        err = float(((z0.float() - ref).abs() / ref.abs().amax(1, keepdim=True)).max()) if ref is not None else -1
        ok = nd == 0 and (ref is None or err < 1e-2)
        bad += not ok
        print(f"{'OK ' if ok else 'BAD'} M={M} K={K} N={N} {mode}: nondeterministic reps {nd}/10, err {err:.2e}", flush=True)
    # exact deferred LayerNorm (per-warp stage release of the side group, 3 packed ops per 2 elements)
    u = fn.fold_colsum(Ws)
    z0 = fn.layernorm_linear(a, Ws, u, cs, eps=1e-5)
    nd = sum(int(not torch.equal(fn.layernorm_linear(a, Ws, u, cs, eps=1e-5), z0))
             for _ in range(int(os.environ.get("REPS", "10"))))
    mu = af.mean(1, keepdim=True)
    ref = ((af - mu) @ Ws.float().T) * torch.rsqrt(((af - mu) ** 2).mean(1, keepdim=True) + 1e-5) + cs
    err = float(((z0.float() - ref).abs() / ref.abs().amax(1, keepdim=True)).max())
    ok = nd == 0 and err < 1e-2
    bad += not ok
    print(f"{'OK ' if ok else 'BAD'} M={M} K={K} N={N} layernorm_linear: nondeterministic reps {nd}, err {err:.2e}",
          flush=True)
print("STRESS", "PASS" if bad == 0 else f"FAIL ({bad})")
