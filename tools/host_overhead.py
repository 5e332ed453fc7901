"""Host-side cost per decode call (config 2, M = 1): the Python binding end to end, the bare C-ABI
call with pre-marshalled ctypes arguments, and the GPU time per call when the host runs ahead.

    python tools/host_overhead.py
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from synth import device as SD  # noqa: E402

dev = torch.device("cuda", 0)
K, N = 4096, 6144
W, g, _, _ = SD.layer(100, N, K, dev, torch.bfloat16)
Ws = fn.fold_weights(W, g)[0]
for M in (1, 16):
    a = SD.activations(7, M, K, dev, torch.bfloat16)
    z = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    for _ in range(50):
        fn.linear(a, Ws, None, eps=1e-5, out=z)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        fn.linear(a, Ws, None, eps=1e-5, out=z)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    L = fn.lib()
    args = (ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(Ws.data_ptr()), None, M, K, N, 1e-5, 0.5, 0, 0,
            ctypes.c_void_p(z.data_ptr()), 0, None, 0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    f = L.flashnorm_linear_ws
    t3 = time.perf_counter()
    for _ in range(n):
        f(*args)
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"M={M}: python binding {1e6 * (t1 - t0) / n:.1f} us/call host ({1e6 * (t2 - t0) / n:.1f} incl. drain); "
          f"bare C ABI {1e6 * (t4 - t3) / n:.1f} us/call host ({1e6 * (t5 - t3) / n:.1f} incl. drain)", flush=True)
