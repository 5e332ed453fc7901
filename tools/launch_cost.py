"""Per-call cost of the pair kernel on small shapes (launch-bound), eager and in a CUDA graph.
Run once per FN_GEMM2_TILE_ROT value (read once per process) to see what the matched-order
table (a 16 KiB __grid_constant__ parameter) costs per launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
if os.environ.get("FN_LIB_OVERRIDE"):
    fn.lib_path = os.environ["FN_LIB_OVERRIDE"]  # A/B against another build of the library
dev = "cuda"
torch.manual_seed(0)
for (M, K, N) in [(256, 512, 512), (512, 1024, 2048), (2048, 4096, 4096)]:
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    W = (torch.randn(N, K, device=dev) / K ** 0.5).to(torch.bfloat16)
    z = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    f = lambda: fn.linear(a, W, None, mode="rmsnorm", path="gemm", out=z)
    for _ in range(5): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize()
    eager = s.elapsed_time(e) / n * 1e3
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(50): f()
    torch.cuda.synchronize()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    s.record()
    for _ in range(4): g.replay()
    e.record(); torch.cuda.synchronize()
    graph = s.elapsed_time(e) / 200 * 1e3
    print(f"lib={os.path.basename(fn.lib_path)} ROT={os.environ.get('FN_GEMM2_TILE_ROT', 'default')} M={M} K={K} N={N}: eager {eager:.2f} us/call, graph {graph:.2f} us/call", flush=True)
