"""A/B timings of the prefill kernels in ONE process (same clocks): config 3 and config 4 shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
dev = "cuda"
def timed(f, steps=10, warm=3):
    """us per call: `steps` calls captured into one CUDA graph and replayed (no host overhead:
    the config-4 shapes run ~40 us, less than the Python wrapper's per-call cost)."""
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        for _ in range(warm): f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            for _ in range(steps): f()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / steps * 1e3
shapes = [(4096, 4096, 28672), (8192, 8192, 28672), (8192, 8192, 14336), (8192, 8192, 7168)] if len(sys.argv) < 2 else eval(sys.argv[1])
for (M, K, N) in shapes:
    a = SD.activations(1, M, K, dev, torch.bfloat16)
    W, g, b, c = SD.layer(1, N, K, dev, torch.bfloat16, with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(W, g, b, c)
    del W
    z = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    out = []
    ws = torch.zeros(fn.linear_workspace_bytes(M, K, N, "dyt", torch.bfloat16), dtype=torch.uint8, device=dev)
    for mode, wsv, tag in (("rmsnorm", "auto", "rmsnorm"), ("none", "auto", "none"), ("dyt", None, "dyt-prologue"),
                           ("dyt", ws, "dyt-prepass")):
        for path in ("gemm", "gemm1"):
            us = timed(lambda: fn.linear(a, Ws, cs, mode=mode, path=path, out=z, workspace=wsv))
            out.append(f"{tag}/{path}={2*M*K*N/us/1e6:.0f}")
    print(f"M={M} K={K} N={N} TFLOP/s: " + " ".join(out), flush=True)
