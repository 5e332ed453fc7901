"""A/B of the K1 fold_weights variants (FN_FOLD_VARIANT is read once per process: run one process per
variant).  Prints the graph-timed per-call time over rotating W (>= 3x L2) and a checksum of W*, c*
so the variants can be compared bit for bit.

    for v in 0 10 11; do FN_FOLD_VARIANT=$v python tools/ab_fold.py; done
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402


def graph_time(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
        for _ in range(reps):
            f()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


dev = torch.device("cuda", 0)
HBM = float(os.environ.get("HBM_GBS", "6549"))
v = os.environ.get("FN_FOLD_VARIANT", "0")
for (N, K) in ((28672, 4096), (6144, 4096), (57344, 8192)):
    nbuf = max(1, -(-3 * 126 * 2 ** 20 // (2 * N * K * 2)))
    Ls = [SD.layer(3 + i, N, K, dev, torch.bfloat16, with_b=True, with_c=True) for i in range(nbuf)]
    Ws = [torch.empty_like(L[0]) for L in Ls]
    cs = [torch.empty(N, device=dev) for _ in Ls]
    it = [0]

    def f():
        i = it[0] % nbuf
        it[0] += 1
        W, g, b, c = Ls[i]
        fn.fold_weights(W, g, b, c, out=Ws[i], c_out=cs[i])
    us = graph_time(f, reps=max(10, 4 * nbuf))
    byts = 2 * N * K * 2 + 4 * (2 * K + 2 * N)
    ck = int(Ws[0].view(torch.int16).to(torch.int64).sum()) ^ int(cs[0].view(torch.int32).to(torch.int64).sum())
    print(f"variant {v} fold_weights {N}x{K}: {us:.1f} us {byts / us / 1e3:.0f} GB/s "
          f"({byts / us / 1e3 / HBM:.3f} of HBM) checksum {ck}", flush=True)
    del Ls, Ws, cs
