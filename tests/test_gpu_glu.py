"""NEXT-1 on the GPU: FFN with a GLU variant (Figs 3-4; readings c24, c25).

* flashnorm_fold_glu_weights: BIT-EXACT against the fold mirror, interleaved in 128-row blocks
* flashnorm_glu_linear: h * s (the deferred hidden times its output scale) against the
  unoptimized oracle hidden act(x Wg) * (x Wu), row-wise relative error <= 2e-2 (bf16)
* flashnorm_linear_scaled and the whole FFN (two launches) against the oracle FFN output
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2407_09577_b200 as fn  # noqa: E402
from oracle import flashnorm_oracle as O  # noqa: E402
from oracle import fold_mirror as FM  # noqa: E402
from synth import bf16_bits, gen_activations, gen_layer  # noqa: E402
from synth import device as SD  # noqa: E402

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
    if x is None:
        return None
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    if dtype == "bf16":
        t = t.to(torch.bfloat16)
    return t.to(DEV)


def H(t):
    return t.float().cpu().numpy()


def bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def interleave(Wg_rows, Wu_rows):
    """[F, K] x 2 -> [2F, K], gate/up in 128-row blocks (include/flashnorm.h)."""
    F, K = Wg_rows.shape
    out = np.empty((2 * F, K), dtype=Wg_rows.dtype)
    for t in range(F // 128):
        out[256 * t:256 * t + 128] = Wg_rows[128 * t:128 * t + 128]
        out[256 * t + 128:256 * t + 256] = Wu_rows[128 * t:128 * t + 128]
    return out


def _glu_layer(seed, M, K, F, amode="normal"):
    a = gen_activations(seed, M, K, amode, "bf16")
    Wg, g, _, _ = gen_layer(seed, F, K, "bf16")
    Wu, _, _, _ = gen_layer(seed + 1000, F, K, "bf16")
    Wd, _, _, _ = gen_layer(seed + 2000, K, F, "bf16")   # down: [n_out = K, F]
    return a, Wg, Wu, Wd, g


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("F,K", [(128, 64), (384, 1000), (1024, 4096)])
def test_fold_glu_weights_bit_exact(dtype, F, K):
    Wg, g, _, _ = gen_layer(21, F, K, dtype)
    Wu, _, _, _ = gen_layer(22, F, K, dtype)
    Wgu = fn.fold_glu_weights(T(Wg, dtype), T(Wu, dtype), T(g, "f32"))
    torch.cuda.synchronize()
    sg = bf16_bits(Wg) if dtype == "bf16" else Wg
    su = bf16_bits(Wu) if dtype == "bf16" else Wu
    mg, _ = FM.fold_weights(sg, g, None, None, dtype)
    mu, _ = FM.fold_weights(su, g, None, None, dtype)
    want = interleave(mg, mu)
    got = bits(Wgu) if dtype == "bf16" else H(Wgu).view(np.uint32)
    np.testing.assert_array_equal(got, want if dtype == "bf16" else want.view(np.uint32))


@pytest.mark.parametrize("act", ["silu", "relu", "bilinear"])
@pytest.mark.parametrize("M,K,F", [(300, 1024, 1024), (16, 4096, 512), (1, 512, 128), (129, 2048, 896)])
def test_glu_linear_parity(act, M, K, F):
    """M > 128: CTA-pair kernel; M <= 128: 1-CTA kernel; h*s vs the unoptimized hidden."""
    a, Wg, Wu, Wd, g = _glu_layer(5, M, K, F)
    Wgu = fn.fold_glu_weights(T(Wg), T(Wu), T(g, "f32"))
    h, s = fn.glu_linear(T(a), Wgu, eps=1e-5, act=act)
    torch.cuda.synchronize()
    ref = O.glu_hidden(a, Wg.T, Wu.T, g, 1e-5, act)
    got = H(h) * H(s)[:, None]
    assert O.rowwise_rel_err(got, ref) <= TOL_BF16
    # the output scale itself: s = r (SwiGLU) or r^2 (ReGLU / bilinear), r = 1/RMSe
    r = 1.0 / O.rmse(a, 1e-5)
    np.testing.assert_allclose(H(s), r if act == "silu" else r * r, rtol=2e-6)


@pytest.mark.parametrize("act", ["silu", "relu"])
def test_glu_ffn_end_to_end(act):
    """y = (h W_down) * s through flashnorm_linear_scaled == the oracle FFN (Fig 3(a)/4(a))."""
    M, K, F = 200, 1024, 768
    a, Wg, Wu, Wd, g = _glu_layer(8, M, K, F, amode="outlier")
    Wgu = fn.fold_glu_weights(T(Wg), T(Wu), T(g, "f32"))
    y = fn.glu_ffn(T(a), Wgu, T(Wd), eps=1e-5, act=act)
    torch.cuda.synchronize()
    ref = O.glu_ffn(a, Wg.T, Wu.T, Wd.T, g, 1e-5, act)
    assert O.rowwise_rel_err(H(y), ref) <= TOL_BF16


@pytest.mark.parametrize("M,K,N", [(1, 1024, 512), (16, 512, 6144), (300, 768, 1000)])
def test_linear_scaled_parity(M, K, N):
    """decode (tcgen05 split-K) and GEMM paths with a given per-row output scale"""
    a = gen_activations(9, M, K, "normal", "bf16")
    Wt, _, _, c = gen_layer(9, N, K, "bf16", with_c=True)
    s = np.linspace(0.25, 4.0, M).astype(np.float32)
    z = fn.linear_scaled(T(a), T(Wt), T(s, "f32"), c_star=T(c, "f32"))
    torch.cuda.synchronize()
    ref = O.linear(a, Wt.T) * s[:, None] + c[None, :]
    assert O.rowwise_rel_err(H(z), ref) <= TOL_BF16


@pytest.mark.parametrize("M,K,N", [(2304, 8192, 2560), (4096, 14336, 4096)])
def test_linear_scaled_stream_k_tail(M, K, N):
    """K >= 8192: the down projection runs the stream-K tail by default (workspace "auto"): rows of
    every 256-row M block against the fp64 oracle, deterministic across launches, and within
    tolerance of the whole-tile kernel (workspace=None)."""
    a = SD.activations(17, M, K, DEV, torch.bfloat16)
    Wt, _, _, c = SD.layer(17, N, K, DEV, torch.bfloat16, with_c=True)
    s = torch.linspace(0.25, 4.0, M, device=DEV, dtype=torch.float32)
    assert fn.linear_workspace_bytes(M, K, N, "none", torch.bfloat16) > 4096  # stream-K scratch planned
    z = fn.linear_scaled(a, Wt, s, c_star=c)
    z2 = fn.linear_scaled(a, Wt, s, c_star=c)
    zw = fn.linear_scaled(a, Wt, s, c_star=c, workspace=None)
    torch.cuda.synchronize()
    assert torch.equal(z, z2)
    rows = np.unique(np.concatenate([np.arange(0, M, 256), np.arange(255, M, 256), [M - 1]]))
    ah = H(a)[rows]
    ref = O.linear(ah, H(Wt).T) * H(s)[rows][:, None] + H(c)[None, :]
    assert O.rowwise_rel_err(H(z)[rows], ref) <= TOL_BF16
    assert O.rowwise_rel_err(H(z), H(zw).astype(np.float64)) <= 1e-2


def test_glu_config3_ffn_full_size_sampled():
    """Llama-3-8B FFN at config 3: M = K = 4096, F = 14336 (gate||up = 28672) — sampled rows"""
    M, K, F = 4096, 4096, 14336
    a = SD.activations(3, M, K, DEV, torch.bfloat16)
    Wg, g, _, _ = SD.layer(31, F, K, DEV, torch.bfloat16)
    Wu, _, _, _ = SD.layer(32, F, K, DEV, torch.bfloat16)
    Wgu = fn.fold_glu_weights(Wg, Wu, g)
    h, s = fn.glu_linear(a, Wgu, eps=1e-5, act="silu")
    torch.cuda.synchronize()
    rows = np.array([0, 1, 777, 2048, 4095])
    ah = H(a)[rows]
    got = H(h[rows]) * H(s)[rows][:, None]
    ref = np.empty_like(got)
    for j0 in range(0, F, 2048):
        j1 = j0 + 2048
        ref[:, j0:j1] = O.glu_hidden(ah, H(Wg[j0:j1]).T, H(Wu[j0:j1]).T, H(g), 1e-5, "silu")
    assert O.rowwise_rel_err(got, ref) <= TOL_BF16
    # deterministic across launches
    h2, _ = fn.glu_linear(a, Wgu, eps=1e-5, act="silu")
    assert torch.equal(h, h2)


def test_glu_validation():
    a = torch.zeros(4, 64, dtype=torch.bfloat16, device=DEV)
    W = torch.zeros(2 * 100, 64, dtype=torch.bfloat16, device=DEV)   # F = 100: not a multiple of 128
    with pytest.raises(fn.FlashNormError, match="multiple of 128"):
        fn.glu_linear(a, W)
    Wg = torch.zeros(100, 64, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(fn.FlashNormError, match="multiple of 128"):
        fn.fold_glu_weights(Wg, Wg)


@pytest.mark.parametrize("M,K,F", [(300, 1024, 1000), (8, 512, 256)])
def test_relu_ffn_end_to_end(M, K, F):
    """Fig 2(b): h = relu(a W*_up) unscaled, s = 1/RMSe(a); y = (h W_down) * s == oracle Fig 2(a)"""
    a = gen_activations(13, M, K, "normal", "bf16")
    Wu, g, _, _ = gen_layer(13, F, K, "bf16")
    Wd, _, _, _ = gen_layer(14, K, F, "bf16")
    Wus, _ = fn.fold_weights(T(Wu), T(g, "f32"))
    h, s = fn.relu_ffn_up(T(a), Wus, eps=1e-5)
    y = fn.linear_scaled(h, T(Wd), s)
    torch.cuda.synchronize()
    assert np.all(H(h) >= 0)
    np.testing.assert_allclose(H(s), 1.0 / O.rmse(a, 1e-5), rtol=2e-6)
    assert O.rowwise_rel_err(H(y), O.relu_ffn(a, Wu.T, Wd.T, g, 1e-5)) <= TOL_BF16
