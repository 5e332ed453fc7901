"""NEXT-2 on the GPU: Q/K/V projection with RoPE (Fig 5(b); readings c26, c27).

The CUDA path (cos/sin scaled by 1/RMS once per token inside the epilogue) against the
unfused oracle Fig 5(a) (RMSNorm -> Q/K/V linear -> RoPE per head, times qk_scale):
row-wise relative error <= 2e-2 (bf16), decode (tcgen05 split-K) and prefill (tcgen05 GEMM).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2407_09577_b200 as fn  # noqa: E402
from oracle import flashnorm_oracle as O  # noqa: E402
from synth import gen_activations, gen_layer  # noqa: E402

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2407_09577_b200 import build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    fn.lib()


def T(x, dtype="bf16"):
    if dtype == "i32":
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).to(DEV)
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    if dtype == "bf16":
        t = t.to(torch.bfloat16)
    return t.to(DEV)


def H(t):
    return t.float().cpu().numpy()


def tables(max_pos, h, base=500000.0):
    i = np.arange(h // 2)
    theta = base ** (-2.0 * i / h)
    ang = np.arange(max_pos)[:, None] * theta[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def run_case(M, K, h, n_q_heads, n_kv_heads, qk_scale, seed=3, max_pos=8192):
    n_rope = (n_q_heads + n_kv_heads) * h
    N = n_rope + n_kv_heads * h
    a = gen_activations(seed, M, K, "normal", "bf16")
    Wt, g, _, _ = gen_layer(seed, N, K, "bf16")
    cos_tab, sin_tab = tables(max_pos, h)
    pos = np.random.default_rng(seed).integers(0, max_pos, M).astype(np.int32)
    Ws, _ = fn.fold_weights(T(Wt), T(g.astype(np.float32), "f32"))
    z = fn.qkv_rope_linear(T(a), Ws, n_rope, h, T(pos, "i32"), T(cos_tab, "f32"), T(sin_tab, "f32"),
                           qk_scale=qk_scale, eps=1e-5)
    torch.cuda.synchronize()
    ref = O.qkv_rope_unfused(a, Wt.T, g, 1e-5, n_rope, h, pos, cos_tab, sin_tab, qk_scale)
    return H(z), ref


@pytest.mark.parametrize("M,nq,nkv", [(3, 144, 8)])
def test_qkv_rope_decode_tall_tiles(M, nq, nkv):
    """N = 20480 > 128 x #SMs: the decode kernel's 256-row tiles (R = 2) also rotate"""
    z, ref = run_case(M, 512, 128, nq, nkv, 1.0)
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16


@pytest.mark.parametrize("M", [1, 16])
def test_qkv_rope_decode_llama3_8b(M):
    """config 2 shape: 4096 -> 32 Q heads + 8 K heads + 8 V heads of 128 (N = 6144)"""
    z, ref = run_case(M, 4096, 128, 32, 8, 1.0 / math.sqrt(math.sqrt(128.0)))
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16


@pytest.mark.parametrize("M", [17, 32, 64, 128])
def test_qkv_rope_batched_decode_llama3_8b(M):
    """config 2 shape at 17..128 tokens: the batched-decode kernel (K4w) rotates Q/K in its epilogue"""
    z, ref = run_case(M, 4096, 128, 32, 8, 1.0 / math.sqrt(math.sqrt(128.0)))
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16


@pytest.mark.parametrize("M,K,h,nq,nkv", [(300, 1024, 64, 8, 2), (64, 512, 128, 4, 4), (257, 2048, 128, 16, 4)])
@pytest.mark.parametrize("qk_scale", [1.0, 0.5])
def test_qkv_rope_prefill(M, K, h, nq, nkv, qk_scale):
    z, ref = run_case(M, K, h, nq, nkv, qk_scale)
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16


def test_qkv_rope_position_zero_is_plain_flashnorm():
    """at position 0 RoPE is the identity: equals flashnorm_linear (rmsnorm) times qk_scale on Q/K"""
    M, K, h = 8, 512, 64
    N = 3 * 2 * h
    a = gen_activations(4, M, K, "normal", "bf16")
    Wt, g, _, _ = gen_layer(4, N, K, "bf16")
    Ws, _ = fn.fold_weights(T(Wt), T(g.astype(np.float32), "f32"))
    cos_tab, sin_tab = tables(4, h)
    z = fn.qkv_rope_linear(T(a), Ws, 4 * h, h, torch.zeros(M, dtype=torch.int32, device=DEV),
                           T(cos_tab, "f32"), T(sin_tab, "f32"), qk_scale=1.0)
    zl = fn.linear(T(a), Ws, eps=1e-5)
    assert torch.equal(z, zl)


def test_qkv_rope_validation():
    a = torch.zeros(4, 64, dtype=torch.bfloat16, device=DEV)
    W = torch.zeros(192, 64, dtype=torch.bfloat16, device=DEV)
    p = torch.zeros(4, dtype=torch.int32, device=DEV)
    c = torch.zeros(4, 32, dtype=torch.float32, device=DEV)
    with pytest.raises(fn.FlashNormError, match="n_rope"):
        fn.qkv_rope_linear(a, W, 100, 64, p, c, c)
    with pytest.raises(fn.FlashNormError, match="head_dim"):
        fn.qkv_rope_linear(a, W, 128, 63, p, c, c)


# ---------------------------------------------------------------- QK-norm + RoPE (NEXT-4 part)

def run_qkn(M, K, h, nq_heads, nk_heads, eps_qk, seed=5, max_pos=4096):
    n_q, n_k = nq_heads * h, nk_heads * h
    N = n_q + n_k + nk_heads * h
    a = gen_activations(seed, M, K, "normal", "bf16")
    Wt, g, _, _ = gen_layer(seed, N, K, "bf16")
    rng = np.random.default_rng(seed)
    g_q = rng.uniform(0.5, 1.5, h).astype(np.float32)
    g_k = rng.uniform(0.5, 1.5, h).astype(np.float32)
    cos_tab, sin_tab = tables(max_pos, h)
    pos = rng.integers(0, max_pos, M).astype(np.int32)
    Ws, _ = fn.fold_weights(T(Wt), T(g.astype(np.float32), "f32"))
    z = fn.qk_norm_rope_linear(T(a), Ws, n_q, n_k, h, T(g_q, "f32"), T(g_k, "f32"), T(pos, "i32"),
                               T(cos_tab, "f32"), T(sin_tab, "f32"), eps_qk=eps_qk, qk_scale=0.5, eps=1e-5)
    torch.cuda.synchronize()
    ref = O.qk_norm_rope_unfused(a, Wt.T, g, 1e-5, n_q, n_k, h, g_q, g_k, eps_qk, pos, cos_tab, sin_tab, 0.5)
    return H(z), ref


@pytest.mark.parametrize("M,K,h,nq,nk", [(1, 2048, 64, 16, 4), (16, 1024, 128, 8, 2), (5, 512, 32, 8, 8),
                                         (300, 1024, 64, 8, 2), (100, 768, 128, 4, 4), (40, 512, 256, 2, 2),
                                         (17, 1024, 32, 8, 8), (64, 2048, 64, 16, 4), (128, 4096, 128, 32, 8)])
@pytest.mark.parametrize("eps_qk", [0.0, 1e-6])
def test_qk_norm_rope_parity(M, K, h, nq, nk, eps_qk):
    """decode (tcgen05 split-K, h | 128), batched decode (17..128 tokens, h | 128) and GEMM paths vs
    the unfused Figs 6(a)+7(a)"""
    z, ref = run_qkn(M, K, h, nq, nk, eps_qk)
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16
