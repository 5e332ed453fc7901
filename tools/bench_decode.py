"""Quick decode (config 2) timing: M in {1,4,16}, K=4096, N=6144, 8 rotating W* buffers (>= 3x L2).
Timed both as eager launches (includes Python/ctypes launch cost) and as a CUDA graph replay."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
dev = "cuda"
K, N = 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 6144
MODE = sys.argv[2] if len(sys.argv) > 2 else "rmsnorm"
NB = max(8, -(-3 * 126 * 2 ** 20 // (K * N * 2)))
Wd = []
for r in range(NB):
    w, g, _, _ = SD.layer(100 + r, N, K, dev, torch.bfloat16)
    Wd.append(fn.fold_weights(w, g)[0])
R = 200
for M in tuple(int(x) for x in os.environ.get("DECODE_MS", "1,4,16").split(",")):
    a = SD.activations(7, M, K, dev, torch.bfloat16)
    z = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    for i in range(20):
        fn.linear(a, Wd[i % NB], None, out=z, mode=MODE)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(R):
        fn.linear(a, Wd[i % NB], None, out=z, mode=MODE)
    e.record(); torch.cuda.synchronize()
    us_eager = s.elapsed_time(e) / R * 1e3
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        fn.linear(a, Wd[0], None, out=z, mode=MODE)
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=st):
            for i in range(R):
                fn.linear(a, Wd[i % NB], None, out=z, mode=MODE)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    s.record()
    gr.replay()
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) / R * 1e3
    byts = K * N * 2 + M * K * 2 + M * N * 2
    print(f"decode {MODE} M={M} N={N}: eager {us_eager:.2f} us ({byts/us_eager/1e3:.0f} GB/s) | graph {us:.2f} us ({byts/us/1e3:.0f} GB/s)", flush=True)
