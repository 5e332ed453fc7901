"""Is the decode time (config 2, graph of 200 PDL-chained calls) sensitive to where the 4 W* buffers
land in HBM?  Re-allocates them behind dummy buffers of varying size in one process."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
dev = "cuda"
W0 = [fn.fold_weights(*SD.layer(100 + i, 6144, 4096, dev, torch.bfloat16)[:2])[0] for i in range(4)]
ad = SD.activations(7, 1, 4096, dev, torch.bfloat16)
zd = torch.empty(1, 6144, dtype=torch.bfloat16, device=dev)
def run(Wd):
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        fn.linear(ad, Wd[0], None, out=zd); torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=st):
            for i in range(200): fn.linear(ad, Wd[i % 4], None, out=zd)
    gr.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        s.record(); gr.replay(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 200 * 1e3)
    return ts
keep = []
for off_mb in (0, 1, 2, 3, 5, 8, 13, 21, 34, 55):
    pad = torch.empty(off_mb * (1 << 20) + 4096, dtype=torch.uint8, device=dev)
    Wd = [w.clone() for w in W0]
    ts = run(Wd)
    print(f"pad {off_mb:3d} MB  W0 @ {Wd[0].data_ptr() % (1 << 30) >> 20:5d} MB (mod 1 GiB): " + " ".join(f"{t:.2f}" for t in ts), flush=True)
    keep.append((pad, Wd))
