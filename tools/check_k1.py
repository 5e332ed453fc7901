"""Bit-exact check of the K1 variant selected by FN_FOLD_VARIANT against the fold mirror, on ragged
shapes and both storage dtypes (tests/test_gpu_parity.py covers the default variant)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09577_b200 as fn  # noqa: E402
from oracle import fold_mirror as FM  # noqa: E402
from synth import bf16_bits, gen_layer  # noqa: E402

v = os.environ.get("FN_FOLD_VARIANT", "0")
ok = True
for dtype in ("bf16", "f32"):
    for (N, K) in ((8, 8), (40, 64), (100, 72), (33, 1000), (5000, 520), (300, 4096), (17, 8192), (20000, 264)):
        for wb in (True, False):
            Wt, g, b, c = gen_layer(21, N, K, dtype, with_b=wb, with_c=True)
            t = torch.from_numpy(np.ascontiguousarray(Wt, np.float32))
            Wd = (t.to(torch.bfloat16) if dtype == "bf16" else t).cuda()
            Ws, cs = fn.fold_weights(Wd, torch.from_numpy(g).cuda(), None if b is None else torch.from_numpy(b).cuda(),
                                     torch.from_numpy(c).cuda())
            Wm, cm = FM.fold_weights(bf16_bits(Wt) if dtype == "bf16" else Wt, g, b, c, dtype)
            got = Ws.view(torch.int16).cpu().numpy().view(np.uint16) if dtype == "bf16" else Ws.cpu().numpy().view(np.uint32)
            okw = np.array_equal(got, Wm if dtype == "bf16" else Wm.view(np.uint32))
            okc = np.array_equal(cs.cpu().numpy().view(np.uint32), cm.view(np.uint32))
            if not (okw and okc):
                print(f"variant {v} {dtype} {N}x{K} b={wb}: W* {'ok' if okw else 'DIFF'} c* {'ok' if okc else 'DIFF'}")
            ok &= okw and okc
print(f"variant {v}: {'BIT-EXACT' if ok else 'MISMATCH'}")
