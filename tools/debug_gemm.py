"""Debug helper: locate wrong tiles of the tcgen05 GEMM against a torch fp32 GPU reference."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
M, K, N = map(int, sys.argv[1:4]); mode = sys.argv[4] if len(sys.argv) > 4 else "rmsnorm"
dev = "cuda"
a = SD.activations(0, M, K, dev, torch.bfloat16)
Wt, g, b, c = SD.layer(0, N, K, dev, torch.bfloat16, with_b=True, with_c=True)
Ws, cs = fn.fold_weights(Wt, g, b, c)
z = fn.linear(a, Ws, cs, eps=1e-5, mode=mode, path="gemm").float()
z2 = fn.linear(a, Ws, cs, eps=1e-5, mode=mode, path="gemm").float()
af = a.float()
acc = af @ Ws.float().T
if mode == "rmsnorm":
    r = torch.rsqrt((af * af).mean(1, keepdim=True) + 1e-5)
    ref = acc * r + cs
else:
    ref = acc + cs
err = (z - ref).abs() / ref.abs().amax(1, keepdim=True)
print(f"[FN_DEBUG={os.environ.get('FN_DEBUG','0')} {mode}] M={M} K={K} N={N}: max err {err.max().item():.3e}; deterministic={torch.equal(z, z2)}")
te = err.view((M + 127) // 128, 128, N // 256, 256).amax(dim=(1, 3)) if M % 128 == 0 and N % 256 == 0 else None
if te is not None:
    bad = (te > 1e-2).nonzero()
    print("bad tiles (m_blk, n_blk):", bad.shape[0], "of", te.numel(), bad[:20].tolist())
    if bad.shape[0]:
        mb, nb = bad[0].tolist()
        sl = (slice(mb * 128, mb * 128 + 128), slice(nb * 256, nb * 256 + 256))
        e = err[sl]
        print("rows bad in tile:", (e.amax(1) > 1e-2).sum().item(), "cols bad:", (e.amax(0) > 1e-2).sum().item())
        ratio = (z[sl] - cs[sl[1]]) / (ref[sl] - cs[sl[1]])
        med = ratio.median(1).values
        print("ratio z/ref per row median: max|dev| %.2e, rows with |dev|>1e-3: %d" % ((med-1).abs().max().item(), ((med-1).abs() > 1e-3).sum().item()))
        print("ratio spread per row (first 8):", (ratio.quantile(0.9, 1) - ratio.quantile(0.1, 1))[:8].tolist())
