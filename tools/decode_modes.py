import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
dev = "cuda"
Wd = [fn.fold_weights(*SD.layer(100 + i, 6144, 4096, dev, torch.bfloat16)[:2])[0] for i in range(4)]
for M in (1, 16):
    ad = SD.activations(7, M, 4096, dev, torch.bfloat16)
    zd = torch.empty(M, 6144, dtype=torch.bfloat16, device=dev)
    for mode in ("rmsnorm", "dyt"):
        st = torch.cuda.Stream(); gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            fn.linear(ad, Wd[0], None, mode=mode, out=zd); torch.cuda.synchronize()
            with torch.cuda.graph(gr, stream=st):
                for i in range(200): fn.linear(ad, Wd[i % 4], None, mode=mode, out=zd)
        gr.replay(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); gr.replay(); e.record(); torch.cuda.synchronize()
        print(f"decode {mode} M={M}: {s.elapsed_time(e) / 200 * 1e3:.2f} us", flush=True)
