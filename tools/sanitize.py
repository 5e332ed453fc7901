"""Every library kernel once, at small ragged shapes, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool synccheck python tools/sanitize.py
    compute-sanitizer --tool initcheck python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py "linear rmsnorm gemm"   (a subset: slow)

Covers: K1 fold_weights (+GLU interleave), K1u fold_colsum, K2 fold_mean_center (3 kernels),
K3 pair + 1-CTA GEMM (rmsnorm, layernorm-exact, dyt prologue and pre-pass, none, GLU, ReLU FFN,
RoPE, QK-norm), K4 tcgen05 decode (rmsnorm, dyt, RoPE, QK-norm) and the mma.sync decode kernel,
K5 fp32, K6 unfused norm, K7 gather permute.  Prints one line per call; exits non-zero on a
library error (the sanitizer reports its own findings)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

dev = "cuda"
bf = torch.bfloat16


ONLY = sys.argv[1] if len(sys.argv) > 1 else None  # substring filter (racecheck is slow)


def run(name, f):
    if ONLY is not None and ONLY not in name:
        return
    f()
    torch.cuda.synchronize()
    print(f"ok {name}", flush=True)


def main():
    M, K, N = 136, 200, 264          # ragged: not multiples of the 128/256 tiles or 64-wide k blocks
    a = SD.activations(1, M, K, dev, bf)
    W, g, b, c = SD.layer(1, N, K, dev, bf, with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(W, g, b, c)
    run("fold_weights", lambda: fn.fold_weights(W, g, b, c))
    run("fold_colsum", lambda: fn.fold_colsum(Ws))
    _, Vt, bp = SD.upstream(1, 8, K, 72, dev, bf)
    run("fold_mean_center", lambda: fn.fold_mean_center(Vt, bp))
    u = fn.fold_colsum(Ws)
    ws = torch.zeros(fn.linear_workspace_bytes(M, K, N, "dyt", torch.bfloat16), dtype=torch.uint8, device=dev)
    for path in ("gemm", "gemm1"):
        for mode in ("rmsnorm", "none", "dyt"):
            run(f"linear {mode} {path}", lambda: fn.linear(a, Ws, cs, mode=mode, path=path))
        run(f"linear dyt prepass {path}", lambda: fn.linear(a, Ws, cs, mode="dyt", path=path, workspace=ws))
    run("layernorm_linear pair", lambda: fn.layernorm_linear(a, Ws, u, cs))
    run("layernorm_linear 1-CTA", lambda: fn.layernorm_linear(a[:40], Ws, u, cs))
    for Md in (1, 5, 16):
        ad = a[:Md].contiguous()
        for mode in ("rmsnorm", "dyt", "none"):
            run(f"decode {mode} M={Md}", lambda: fn.linear(ad, Ws, cs, mode=mode, path="gemv"))
        run(f"decode mma.sync M={Md}", lambda: fn.linear(ad, Ws, cs, path="gemv_mma"))
    F = 256
    Wg, gg, _, _ = SD.layer(2, F, K, dev, bf)
    Wu, _, _, _ = SD.layer(3, F, K, dev, bf)
    Wgu = fn.fold_glu_weights(Wg, Wu, gg)
    Wd, _, _, _ = SD.layer(4, K, F, dev, bf)
    for act in ("silu", "relu", "bilinear"):
        run(f"glu {act}", lambda: fn.glu_ffn(a, Wgu, Wd, act=act))
    run("relu_ffn_up", lambda: fn.relu_ffn_up(a, Ws))
    h, hd = 64, 32
    pos = torch.arange(M, dtype=torch.int32, device=dev)
    inv = 1.0 / (10000 ** (torch.arange(0, hd, dtype=torch.float32, device=dev) / h))
    ang = torch.arange(M, dtype=torch.float32, device=dev)[:, None] * inv[None, :]
    cos, sin = torch.cos(ang).contiguous(), torch.sin(ang).contiguous()
    Wq, gq, _, _ = SD.layer(5, 384, K, dev, bf)
    Wqs, _ = fn.fold_weights(Wq, gq)
    gqn = torch.ones(h, dtype=torch.float32, device=dev)
    for Mq in (M, 3):
        aq = a[:Mq].contiguous()
        run(f"qkv_rope M={Mq}", lambda: fn.qkv_rope_linear(aq, Wqs, 256, h, pos[:Mq], cos, sin))
        run(f"qk_norm_rope M={Mq}", lambda: fn.qk_norm_rope_linear(aq, Wqs, 128, 128, h, gqn, gqn, pos[:Mq], cos,
                                                                    sin))
    a32 = a.float()
    W32, g32, _, _ = SD.layer(6, 72, K, dev, torch.float32)
    Ws32, cs32 = fn.fold_weights(W32, g32)
    for mode in ("rmsnorm", "dyt", "none"):
        run(f"f32 {mode}", lambda: fn.linear(a32, Ws32, cs32, mode=mode))
    run("f32 layernorm_linear", lambda: fn.layernorm_linear(a32, Ws32, fn.fold_colsum(Ws32), cs32))
    run("baseline_norm", lambda: fn.baseline_norm(a, g, b))
    parts = torch.randn(2, M, 64, device=dev).to(bf)
    run("gather_columns", lambda: fn.gather_columns(parts))
    print("sanitize: all calls returned", flush=True)


if __name__ == "__main__":
    main()
