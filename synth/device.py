"""Seeded synthetic inputs generated directly on the GPU (full BASELINE sizes).

Same recipe as synth/inputs.py, drawn with
torch's Philox generator on the device so that multi-GB weights do not have to
be generated on the host.  No FlashNorm arithmetic here.  Parity tests copy the
sampled operands back to the host for the oracle, so both sides still see the
identical bits.
"""
from __future__ import annotations

import math

from .inputs import TENSOR_IDS


def _gen(seed: int, name: str, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 1_000_003 + TENSOR_IDS[name])
    return g


def normal(seed, name, shape, device, dtype, std=1.0, mean=0.0):
    import torch
    x = torch.randn(shape, generator=_gen(seed, name, device), device=device, dtype=torch.float32)
    if std != 1.0:
        x.mul_(std)
    if mean != 0.0:
        x.add_(mean)
    return x.to(dtype)  # RNE


def uniform(seed, name, shape, device, dtype, lo, hi):
    import torch
    x = torch.rand(shape, generator=_gen(seed, name, device), device=device, dtype=torch.float32)
    return (x * (hi - lo) + lo).to(dtype)


def layer(seed, N, K, device, dtype, with_g=True, with_b=False, with_c=False):
    """Wt[N,K] ~ N(0, 1/K); g ~ U[0.5,1.5]; b, c ~ U[-0.1, 0.1] (fp32 vectors)."""
    import torch
    Wt = normal(seed, "W", (N, K), device, dtype, std=1.0 / math.sqrt(K))
    g = uniform(seed, "g", (K,), device, torch.float32, 0.5, 1.5) if with_g else None
    b = uniform(seed, "b", (K,), device, torch.float32, -0.1, 0.1) if with_b else None
    c = uniform(seed, "c", (N,), device, torch.float32, -0.1, 0.1) if with_c else None
    return Wt, g, b, c


def activations(seed, M, K, device, dtype, name="a"):
    """a[M,K] ~ N(0,1)."""
    return normal(seed, name, (M, K), device, dtype)


def upstream(seed, M, d_in, n_out, device, dtype):
    """x[M,d_in] ~ N(0,1); Vt[n_out,d_in] with per-input-row mean mu_i ~ U[-0.05,0.05]; b_prev ~ U[-0.5,1.5]."""
    import torch
    x = activations(seed, M, d_in, device, dtype, name="x")
    mu = uniform(seed + 7919, "V", (1, d_in), device, torch.float32, -0.05, 0.05)
    Vt = (torch.randn((n_out, d_in), generator=_gen(seed, "V", device), device=device, dtype=torch.float32)
          .mul_(1.0 / math.sqrt(d_in)).add_(mu)).to(dtype)
    b_prev = uniform(seed, "b_prev", (n_out,), device, torch.float32, -0.5, 1.5)
    return x, Vt, b_prev
