"""Timings for every BASELINE.json config (one GPU), printed as JSON lines + a markdown table.

    python tools/bench_configs.py [--quick]

Config 1 tiny fp32 (latency), 2 decode (GB/s), 3 prefill (TFLOP/s), 4 LayerNorm
retrofit (V fold, upstream V* GEMM, LN linear) and DyT at N=4096/16384, 5 Llama-3-70B
FFN shapes (P=1 and the per-rank shard of P=2/4/8), and the folds.  Inputs larger
than L2 or rotated; CUDA events on the launching stream; small kernels timed as a
CUDA graph of back-to-back calls.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

dev = torch.device("cuda", 0)
PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
TF, HBM = PEAKS["bf16_tflops"], PEAKS["hbm_gbs"]
QUICK = "--quick" in sys.argv
rows = []


def timed(f, steps, warm=3, graph=False):
    for _ in range(warm):
        f(0)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph:
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
            for i in range(steps):
                f(i)
        g.replay()
        torch.cuda.synchronize()
        s.record()
        g.replay()
        e.record()
    else:
        s.record()
        for i in range(steps):
            f(i)
        e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps * 1e3  # us


def report(config, what, us, flops=None, byts=None):
    r = {"config": config, "what": what, "us": round(us, 3)}
    if flops:
        r["TFLOP/s"] = round(flops / us / 1e6, 1)
        r["frac_bf16_peak"] = round(flops / us / 1e6 / TF, 3)
    if byts:
        r["GB/s"] = round(byts / us / 1e3, 1)
        r["frac_hbm"] = round(byts / us / 1e3 / HBM, 3)
    rows.append(r)
    print(json.dumps(r), flush=True)


# ---------------- config 1: tiny fp32
a = SD.activations(1, 8, 64, dev, torch.float32)
W, g, b, c = SD.layer(1, 64, 64, dev, torch.float32, with_b=True, with_c=True)
Ws, cs = fn.fold_weights(W, g, b, c)
for mode in ("rmsnorm", "layernorm", "dyt"):
    z = torch.empty(8, 64, device=dev)
    us = timed(lambda i: fn.linear(a, Ws, cs, mode=mode, out=z), 200, graph=True)
    report("1 tiny fp32 M=8 K=64 N=64", f"linear {mode} (per call, graph)", us, flops=2 * 8 * 64 * 64)

# ---------------- config 2: decode
K, N = 4096, 6144
Wd = []
for r in range(4):
    w, gg, _, _ = SD.layer(100 + r, N, K, dev, torch.bfloat16)
    Wd.append(fn.fold_weights(w, gg)[0])
    del w
for M in (1, 16):
    ad = SD.activations(7, M, K, dev, torch.bfloat16)
    zd = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    for mode, path in (("rmsnorm", "auto"), ("dyt", "auto"), ("rmsnorm", "gemv_mma")):
        us = timed(lambda i: fn.linear(ad, Wd[i % 4], None, mode=mode, path=path, out=zd), 200, graph=True)
        report(f"2 decode M={M} K=4096 N=6144", f"linear {mode} path={path} (graph, 4 rotating W*)", us,
               byts=K * N * 2 + M * K * 2 + M * N * 2)
# NEXT-2: the same QKV projection with RoPE fused (32 Q + 8 K heads of 128 rotated, V plain)
i_ = torch.arange(64, device=dev, dtype=torch.float64)
ang = torch.arange(8192, device=dev, dtype=torch.float64)[:, None] * (500000.0 ** (-2.0 * i_ / 128))[None, :]
cos_t, sin_t = torch.cos(ang).float(), torch.sin(ang).float()
for M in (1, 16):
    ad = SD.activations(7, M, K, dev, torch.bfloat16)
    zd = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    posd = torch.arange(M, device=dev, dtype=torch.int32) + 1000
    us = timed(lambda i: fn.qkv_rope_linear(ad, Wd[i % 4], 5120, 128, posd, cos_t, sin_t, qk_scale=128 ** -0.25,
                                            out=zd), 200, graph=True)
    report(f"NEXT-2 decode M={M} K=4096 N=6144", "qkv_rope_linear (graph, 4 rotating W*)", us,
           byts=K * N * 2 + M * K * 2 + M * N * 2)
del Wd

# ---------------- config 3: prefill + folds
M, K, N = 4096, 4096, 28672
a = SD.activations(3, M, K, dev, torch.bfloat16)
W, g, b, c = SD.layer(3, N, K, dev, torch.bfloat16, with_b=True, with_c=True)
Ws = torch.empty_like(W)
cs = torch.empty(N, device=dev)
us = timed(lambda i: fn.fold_weights(W, g, b, c, out=Ws, c_out=cs), 5)
report("3 prefill W fold", "fold_weights 28672x4096 (g, b, c)", us, byts=2 * N * K * 2 + 4 * (2 * K + 2 * N))
z = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
for mode, path, wsp in (("rmsnorm", "auto", "auto"), ("none", "auto", "auto"), ("rmsnorm", "gemm1", "auto"),
                        ("dyt", "auto", "auto"), ("dyt", "auto", None)):
    us = timed(lambda i: fn.linear(a, Ws, cs, mode=mode, path=path, out=z, workspace=wsp), 10 if not QUICK else 3)
    tag = " (tanh prologue, no workspace)" if (mode == "dyt" and wsp is None) else (" (K8 pre-pass)" if mode == "dyt" else "")
    report("3 prefill M=4096 K=4096 N=28672", f"linear {mode} path={path}{tag}", us, flops=2 * M * K * N)
# NEXT-2 prefill: the RoPE epilogue on the same GEMM (Q/K = the first 5120 of 28672 columns)
pos3 = (torch.arange(M, device=dev, dtype=torch.int32) % 8192)
us = timed(lambda i: fn.qkv_rope_linear(a, Ws, 5120, 128, pos3, cos_t, sin_t, qk_scale=128 ** -0.25, out=z),
           10 if not QUICK else 3)
report("NEXT-2 prefill M=4096 K=4096 N=28672", "qkv_rope_linear (RoPE on 5120 columns)", us, flops=2 * M * K * N)

# NEXT-1: SwiGLU FFN at config 3 (gate||up with the GLU epilogue + scaled down projection)
F = N // 2
Wgu = fn.fold_glu_weights(Ws[:F], Ws[F:], None)
h = torch.empty((M, F), dtype=torch.bfloat16, device=dev)
sg = torch.empty(M, dtype=torch.float32, device=dev)
for act in ("silu", "relu"):
    us = timed(lambda i: fn.glu_linear(a, Wgu, eps=1e-5, act=act, out=h, s_out=sg), 10 if not QUICK else 3)
    report("NEXT-1 GLU FFN M=4096 K=4096 F=14336", f"glu_linear {act} (gate||up GEMM + GLU epilogue)", us,
           flops=2 * M * K * N)
Wdn, _, _, _ = SD.layer(77, K, F, dev, torch.bfloat16)
yd = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
us = timed(lambda i: fn.linear_scaled(h, Wdn, sg, out=yd), 10 if not QUICK else 3)
report("NEXT-1 GLU FFN M=4096 K=4096 F=14336", "linear_scaled down 14336->4096 (x s)", us, flops=2 * M * F * K)
del Wgu, h, Wdn, yd
del W, Ws, z

# ---------------- config 4: LayerNorm retrofit (V* fold + upstream GEMM + LN linear) and DyT
M, d = 2048, 4096
x, Vt, bp = SD.upstream(4, M, d, d, dev, torch.bfloat16)
Vs0 = torch.empty_like(Vt)
wsv = torch.zeros(fn.fold_mean_center_workspace_bytes(d, d) // 8 + 2, dtype=torch.float64, device=dev)
us = timed(lambda i: fn.fold_mean_center(Vt, bp, out=Vs0, workspace=wsv), 20, graph=True)
report("4 LN V fold", "fold_mean_center 4096x4096 (+b_prev), graph", us, byts=2 * d * d * 2)
del Vs0, wsv
Vs, bs = fn.fold_mean_center(Vt, bp)
astar = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
# config-4 GEMMs run ~45 us: CUDA graphs of back-to-back calls (the Python wrapper's per-call cost
# is of the same order, so eager timing would measure the host)
us = timed(lambda i: fn.linear(x, Vs, bs, mode="none", out=astar), 20, graph=True)
report("4 upstream x V* + b*", "linear none M=2048 K=4096 N=4096 (graph)", us, flops=2 * M * d * d)
for Nout in (4096, 16384):
    W, g, b, c = SD.layer(5, Nout, d, dev, torch.bfloat16, with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(W, g, b, c)
    u = fn.fold_colsum(Ws)
    z = torch.empty(M, Nout, dtype=torch.bfloat16, device=dev)
    for mode in ("layernorm", "rmsnorm", "dyt"):
        us = timed(lambda i: fn.linear(astar, Ws, cs, mode=mode, out=z), 20, graph=True)
        report(f"4 M=2048 K=4096 N={Nout}", f"linear {mode} (graph)", us, flops=2 * M * d * Nout)
    us = timed(lambda i: fn.layernorm_linear(x, Ws, u, cs, eps=1e-5, out=z), 20, graph=True)
    report(f"4 M=2048 K=4096 N={Nout}", "layernorm_linear (exact LN, no V fold; graph)", us, flops=2 * M * d * Nout)
    del W, Ws, z, u

# ---------------- config 5: Llama-3-70B FFN shapes, one rank's shard for P = 1, 2, 4, 8
M, K, Nfull = 8192, 8192, 57344
a = SD.activations(6, M, K, dev, torch.bfloat16)
W, g, _, _ = SD.layer(6, Nfull, K, dev, torch.bfloat16)
Ws, _ = fn.fold_weights(W, g)
del W
for P in ((1, 2, 4, 8) if not QUICK else (1, 8)):
    Nl = Nfull // P
    Wl = Ws[:Nl]
    z = torch.empty(M, Nl, dtype=torch.bfloat16, device=dev)
    us = timed(lambda i: fn.linear(a, Wl, None, out=z), 5 if P < 4 else 10)
    report(f"5 70B FFN M=8192 K=8192 N={Nfull}/P", f"rank shard P={P} (N_local={Nl})", us, flops=2 * M * K * Nl)
    del z

print("\n| config | what | µs | TFLOP/s | of bf16 peak | GB/s | of HBM |")
print("|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r['config']} | {r['what']} | {r['us']} | {r.get('TFLOP/s', '')} | {r.get('frac_bf16_peak', '')} | "
          f"{r.get('GB/s', '')} | {r.get('frac_hbm', '')} |")
