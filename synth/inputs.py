"""Counter-based seeded generators for FlashNorm workloads (no method arithmetic).

Every tensor is drawn from numpy's Philox-4x64 keyed by (seed, tensor_id), so a
tensor is reproducible independently of what else was generated.  Values are
produced in float32 and, for the bf16 path, rounded to bf16 (round-to-nearest-
even) HERE, on the host: the oracle consumes the rounded float values, the GPU
consumes the identical bf16 bit patterns.

Tensor ids: a=1, W=2, g=3, b=4, c=5, V=6, b_prev=7, x=8.

Layouts follow the CUDA boundary: weights are generated in storage layout
``Wt[N, K]`` (nn.Linear layout, K contiguous).  The paper's ``W`` (K x N,
``y = x W``) is ``Wt.T``.
"""
from __future__ import annotations

import numpy as np

TENSOR_IDS = {"a": 1, "W": 2, "g": 3, "b": 4, "c": 5, "V": 6, "b_prev": 7, "x": 8}


def rng(seed: int, tensor_id: int) -> np.random.Generator:
    """Independent Philox stream for (seed, tensor_id)."""
    return np.random.Generator(np.random.Philox(key=(int(seed) << 32) | int(tensor_id)))


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern (uint16), round-to-nearest-even (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounded = u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    return (rounded >> np.uint32(16)).astype(np.uint16)


def bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """bf16 bit pattern (uint16) -> float32 (exact)."""
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 value, returned as float32."""
    return bits_to_f32(bf16_bits(x))


def _finish(x: np.ndarray, dtype: str) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    if dtype == "bf16":
        return bf16_round(x)
    if dtype == "f32":
        return x
    raise ValueError(f"dtype must be 'bf16' or 'f32', got {dtype!r}")


def gen_tensor(seed: int, name: str, shape, dist: str, dtype: str = "bf16", **kw) -> np.ndarray:
    """One seeded tensor. dist: 'normal' (mean, std), 'uniform' (lo, hi)."""
    g = rng(seed, TENSOR_IDS[name])
    if dist == "normal":
        x = g.standard_normal(size=shape, dtype=np.float32) * np.float32(kw.get("std", 1.0))
        x = x + np.float32(kw.get("mean", 0.0))
    elif dist == "uniform":
        x = g.uniform(kw.get("lo", -1.0), kw.get("hi", 1.0), size=shape).astype(np.float32)
    else:
        raise ValueError(dist)
    return _finish(x, dtype)


def gen_activations(seed: int, M: int, K: int, mode: str = "normal", dtype: str = "bf16",
                    name: str = "a") -> np.ndarray:
    """Activations a[M, K].

    normal    : a ~ N(0, 1)
    uniform   : a ~ U[-1, 1] (tiny config)
    outlier   : N(0,1) with 4 fixed channels scaled x200 (Llama massive-activation structure)
    lowenergy : each row scaled by 10^u, u ~ U[-3, 3] -> exercises eps (App. A)
    shifted   : N(0,1) plus a per-row offset ~ U[-3, 3]: LayerNorm inputs with non-zero means
                (the deferred LayerNorm without a foldable V, reading c29)
    """
    g = rng(seed, TENSOR_IDS[name])
    if mode == "uniform":
        x = g.uniform(-1.0, 1.0, size=(M, K)).astype(np.float32)
    else:
        x = g.standard_normal(size=(M, K), dtype=np.float32)
        if mode == "outlier":
            ch = rng(seed, 100 + TENSOR_IDS[name]).choice(K, size=min(4, K), replace=False)
            x[:, ch] *= np.float32(200.0)
        elif mode == "lowenergy":
            u = rng(seed, 200 + TENSOR_IDS[name]).uniform(-3.0, 3.0, size=(M, 1))
            x = (x * np.power(10.0, u)).astype(np.float32)
        elif mode == "shifted":
            off = rng(seed, 300 + TENSOR_IDS[name]).uniform(-3.0, 3.0, size=(M, 1))
            x = (x + off).astype(np.float32)
        elif mode != "normal":
            raise ValueError(mode)
    return _finish(x, dtype)


def gen_layer(seed: int, N: int, K: int, dtype: str = "bf16", *, with_g=True, with_b=False,
              with_c=False, tiny: bool = False):
    """Norm + linear parameters: Wt[N,K] (storage), g[K], b[K], c[N] (fp32 vectors).

    W ~ N(0, 1/K) (tiny: U[-1,1]); g ~ U[0.5, 1.5];
    b, c ~ U[-0.1, 0.1].  Vectors are float32 (the ABI takes fp32 vectors).
    """
    if tiny:
        Wt = gen_tensor(seed, "W", (N, K), "uniform", dtype, lo=-1.0, hi=1.0)
    else:
        Wt = gen_tensor(seed, "W", (N, K), "normal", dtype, std=1.0 / np.sqrt(K))
    g = gen_tensor(seed, "g", (K,), "uniform", "f32", lo=0.5, hi=1.5) if with_g else None
    b = gen_tensor(seed, "b", (K,), "uniform", "f32", lo=-0.1, hi=0.1) if with_b else None
    c = gen_tensor(seed, "c", (N,), "uniform", "f32", lo=-0.1, hi=0.1) if with_c else None
    return Wt, g, b, c


def gen_upstream(seed: int, M: int, d_in: int, n_out: int, dtype: str = "bf16"):
    """Config-4 upstream layer: x[M, d_in], Vt[n_out, d_in] (storage), b_prev[n_out].

    Paper V is d_in x n_out (y = x V); V[i, :] ~ N(mu_i, 1/d_in) with a
    per-input-row mean mu_i ~ U[-0.05, 0.05] so that the row sums s_i are non-zero
    and the mean-centering fold is non-trivial; b_prev ~ U[-0.5, 1.5]
    (non-zero mean, so the b_prev reading c7 matters).
    """
    x = gen_activations(seed, M, d_in, "normal", dtype, name="x")
    g = rng(seed, TENSOR_IDS["V"])
    mu = g.uniform(-0.05, 0.05, size=(1, d_in)).astype(np.float32)
    Vt = g.standard_normal(size=(n_out, d_in), dtype=np.float32) * np.float32(1.0 / np.sqrt(d_in)) + mu
    Vt = _finish(Vt, dtype)
    b_prev = gen_tensor(seed, "b_prev", (n_out,), "uniform", "f32", lo=-0.5, hi=1.5)
    return x, Vt, b_prev
