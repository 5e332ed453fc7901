"""GPU parity: the CUDA path (through the C ABI) against the oracle.

* folds: BIT-EXACT against oracle/fold_mirror.py (same precision and order)
* linear: row-wise inf-norm relative error (reading c12) against the fp64 oracle
  on the same seeded inputs: <= 2e-2 for bf16, <= 1e-5 for f32 (BASELINE.json:5)
* full BASELINE sizes in the launch configuration bench.py times: sampled rows
  against the oracle + size-independent properties (determinism, row
  permutation, column-shard concatenation)
"""
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2407_09577_b200 as fn  # noqa: E402
from oracle import flashnorm_oracle as O  # noqa: E402
from oracle import fold_mirror as FM  # noqa: E402
from synth import bf16_bits, gen_activations, gen_layer, gen_upstream  # noqa: E402
from synth import device as SD  # noqa: E402

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
TOL_F32 = 1e-5
DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2407_09577_b200 import build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    fn.lib()


def T(x, dtype="bf16"):
    """host float32 values (already representable) -> device tensor (exact)."""
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


# ============================================================ folds, bit-exact

GBC = [(1, 1, 1), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (0, 0, 0)]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("N,K", [(8, 8), (64, 64), (13, 1000), (300, 4096), (1031, 2048)])
@pytest.mark.parametrize("gbc", GBC)
def test_fold_weights_bit_exact(dtype, N, K, gbc):
    Wt, g, b, c = gen_layer(11, N, K, dtype, with_b=True, with_c=True)
    g, b, c = (g if gbc[0] else None), (b if gbc[1] else None), (c if gbc[2] else None)
    Ws, cs = fn.fold_weights(T(Wt, dtype), T(g, "f32"), T(b, "f32"), T(c, "f32"))
    torch.cuda.synchronize()
    store = bf16_bits(Wt) if dtype == "bf16" else Wt
    Wm, cm = FM.fold_weights(store, g, b, c, dtype)
    if dtype == "bf16":
        np.testing.assert_array_equal(bits(Ws), Wm)
    else:
        np.testing.assert_array_equal(H(Ws).view(np.uint32), Wm.view(np.uint32))
    if cm is not None:
        np.testing.assert_array_equal(H(cs).view(np.uint32), cm.view(np.uint32))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("n_out,d_in", [(8, 8), (40, 24), (100, 72), (33, 1000), (4096, 4096), (5000, 520),
                                         (20000, 264), (66304, 256), (6144, 4096)])
@pytest.mark.parametrize("with_b", [True, False])
def test_fold_mean_center_bit_exact(dtype, n_out, d_in, with_b):
    _, Vt, bp = gen_upstream(12, 2, d_in, n_out, dtype)
    bp = bp if with_b else None
    Vs, bs = fn.fold_mean_center(T(Vt, dtype), T(bp, "f32"))
    torch.cuda.synchronize()
    store = bf16_bits(Vt) if dtype == "bf16" else Vt
    Vm, bm, _ = FM.fold_mean_center(store, bp, dtype)
    if dtype == "bf16":
        np.testing.assert_array_equal(bits(Vs), Vm)
    else:
        np.testing.assert_array_equal(H(Vs).view(np.uint32), Vm.view(np.uint32))
    if with_b:
        np.testing.assert_array_equal(H(bs).view(np.uint32), bm.view(np.uint32))


_K2_VARIANT = r'''
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_2407_09577_b200 as fn
from oracle import fold_mirror as FM
from synth import gen_upstream, bf16_bits
ok = True
for dtype in ("bf16", "f32"):
    for (n_out, d_in) in [(8, 8), (33, 1000), (100, 72), (4096, 4096), (20000, 264), (7000, 2056)]:
        _, Vt, bp = gen_upstream(12, 2, d_in, n_out, dtype)
        t = torch.from_numpy(np.ascontiguousarray(Vt, dtype=np.float32))
        t = (t.to(torch.bfloat16) if dtype == "bf16" else t).cuda()
        Vs, bs = fn.fold_mean_center(t, torch.from_numpy(bp).cuda())
        torch.cuda.synchronize()
        Vm, bm, _ = FM.fold_mean_center(bf16_bits(Vt) if dtype == "bf16" else Vt, bp, dtype)
        got = Vs.view(torch.int16).cpu().numpy().view(np.uint16) if dtype == "bf16" else Vs.cpu().numpy().view(np.uint32)
        ok &= np.array_equal(got, Vm if dtype == "bf16" else Vm.view(np.uint32))
        ok &= np.array_equal(bs.cpu().numpy().view(np.uint32), bm.view(np.uint32))
print("K2_VARIANT_OK" if ok else "K2_VARIANT_DIFF")
'''


@pytest.mark.parametrize("variant", ["1", "3"])
def test_fold_mean_center_cluster_variant_bit_exact(variant):
    """FN_K2_VARIANT=1: the one-launch cluster kernel (DSMEM reduction, TMA stores) meets the same
    contract bit for bit, including ragged shapes, resident (<= 6 boxes per lane group) and
    streamed (more) slabs, and clusters that loop over several slabs.  FN_K2_VARIANT=3: the
    three-launch kernels (the default's fallback when V does not fit the persistent kernel's
    resident tiles) on the same shapes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _K2_VARIANT, root], env=dict(os.environ, FN_K2_VARIANT=variant),
                       capture_output=True, text=True, timeout=600)
    assert "K2_VARIANT_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_fold_mean_center_workspace_reuse_and_graph_replay(dtype):
    """Back-to-back calls with one caller-owned workspace and replays of a captured CUDA graph whose
    input V changes in place between replays: every result stays bit-exact against the mirror."""
    n_out, d_in = 3000, 1040
    ws = torch.zeros(fn.fold_mean_center_workspace_bytes(n_out, d_in) // 8 + 2, dtype=torch.float64, device=DEV)
    outs = []
    for seed in (13, 14, 15):
        _, Vt, bp = gen_upstream(seed, 2, d_in, n_out, dtype)
        Vs, bs = fn.fold_mean_center(T(Vt, dtype), T(bp, "f32"), workspace=ws)
        torch.cuda.synchronize()
        Vm, bm, _ = FM.fold_mean_center(bf16_bits(Vt) if dtype == "bf16" else Vt, bp, dtype)
        got = bits(Vs) if dtype == "bf16" else H(Vs).view(np.uint32)
        np.testing.assert_array_equal(got, Vm if dtype == "bf16" else Vm.view(np.uint32))
        np.testing.assert_array_equal(H(bs).view(np.uint32), bm.view(np.uint32))
        outs.append(Vt)
    Vin = T(outs[0], dtype)
    Vout = torch.empty_like(Vin)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn.fold_mean_center(Vin, None, out=Vout, workspace=ws)   # warm (descriptor encode, attributes)
        st.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            fn.fold_mean_center(Vin, None, out=Vout, workspace=ws)
    for Vt in outs[1:] + outs[:1]:
        Vin.copy_(T(Vt, dtype))
        graph.replay()
        torch.cuda.synchronize()
        Vm, _, _ = FM.fold_mean_center(bf16_bits(Vt) if dtype == "bf16" else Vt, None, dtype)
        got = bits(Vout) if dtype == "bf16" else H(Vout).view(np.uint32)
        np.testing.assert_array_equal(got, Vm if dtype == "bf16" else Vm.view(np.uint32))


def _special_matrix(rows, cols, dtype, seed=5):
    """Values that stress the exact fp64 fold arithmetic: zero columns, bf16/f32 subnormals,
    huge and tiny magnitudes in one column (rounding in the fp64 sums), +-inf and NaN."""
    rng = np.random.default_rng(seed)
    x = rng.normal(0, 0.02, (rows, cols)).astype(np.float32)
    x[:, 0] = 0.0
    x[:, 1] = -0.0
    x[:, 2] = rng.choice([1e-39, -3e-40, 9.2e-41], rows).astype(np.float32)   # subnormal (bf16 too)
    x[:, 3] = rng.choice([3e38, -2e38, 1e-30, 7.0], rows).astype(np.float32)  # wide exponent range
    x[:, 4] = rng.normal(0, 1, rows).astype(np.float32) * np.float32(2.0 ** 100)
    x[rows // 2, 5] = np.inf
    x[rows // 3, 6] = -np.inf
    x[rows // 4, 7] = np.nan
    if dtype == "bf16":
        from synth import bf16_round
        x = bf16_round(x).astype(np.float32)
    return x


def _bits_equal_nan_aware(got_bits, want_bits, dtype):
    if dtype == "bf16":
        g32 = (got_bits.astype(np.uint32) << 16).view(np.float32)
        w32 = (want_bits.astype(np.uint32) << 16).view(np.float32)
    else:
        g32, w32 = got_bits.view(np.float32), want_bits.view(np.float32)
    nan = np.isnan(w32)
    np.testing.assert_array_equal(np.isnan(g32), nan)
    np.testing.assert_array_equal(got_bits[~nan], want_bits[~nan])


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("n_out", [64, 1000])
def test_fold_mean_center_special_values(dtype, n_out):
    """zeros, subnormals, wide exponent ranges, +-inf, NaN: still bit-exact vs the mirror
    (the K2 kernels widen bf16/f32 to fp64 with integer ops and fall back on inf/NaN)."""
    Vt = _special_matrix(n_out, 1032, dtype)
    bp = np.linspace(-1, 1, n_out).astype(np.float32)
    Vs, bs = fn.fold_mean_center(T(Vt, dtype), T(bp, "f32"))
    torch.cuda.synchronize()
    store = bf16_bits(Vt) if dtype == "bf16" else Vt
    Vm, bm, _ = FM.fold_mean_center(store, bp, dtype)
    got = bits(Vs) if dtype == "bf16" else H(Vs).view(np.uint32)
    _bits_equal_nan_aware(got, Vm if dtype == "bf16" else Vm.view(np.uint32), dtype)
    np.testing.assert_array_equal(H(bs).view(np.uint32), bm.view(np.uint32))


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_fold_weights_special_values(dtype):
    Wt = _special_matrix(1000, 1032, dtype).T.copy()   # [N=1032, K=1000]: specials in rows
    K = Wt.shape[1]
    g = np.linspace(0.5, 1.5, K).astype(np.float32)
    b = np.linspace(-0.1, 0.1, K).astype(np.float32)
    c = np.zeros(Wt.shape[0], np.float32)
    Ws, cs = fn.fold_weights(T(Wt, dtype), T(g, "f32"), T(b, "f32"), T(c, "f32"))
    torch.cuda.synchronize()
    store = bf16_bits(Wt) if dtype == "bf16" else Wt
    Wm, cm = FM.fold_weights(store, g, b, c, dtype)
    got = bits(Ws) if dtype == "bf16" else H(Ws).view(np.uint32)
    _bits_equal_nan_aware(got, Wm if dtype == "bf16" else Wm.view(np.uint32), dtype)
    _bits_equal_nan_aware(H(cs).view(np.uint32), cm.view(np.uint32), "f32")


# ============================================================ linear: f32 path (config 1)

def _layer_and_ref(seed, M, K, N, dtype, mode, amode="normal", eps=1e-5, alpha=0.5, bias=True, tiny=False):
    a = gen_activations(seed, M, K, "uniform" if tiny else amode, dtype)
    if mode == "layernorm":  # input of the LayerNorm-mode kernel is pre-centered (reading c9)
        a = a - a.mean(axis=1, keepdims=True)
        if dtype == "bf16":
            from synth import bf16_round
            a = bf16_round(a.astype(np.float32))
        a = a.astype(np.float32)
    Wt, g, b, c = gen_layer(seed, N, K, dtype, with_b=bias and mode != "none", with_c=bias, tiny=tiny)
    if mode == "none":
        g = None
    ref = O.norm_linear(a, Wt.T, g, b, c, eps, mode, alpha) if mode != "none" else O.linear(a, Wt.T, c)
    return a, Wt, g, b, c, ref


def _run(a, Wt, g, b, c, dtype, mode, eps=1e-5, alpha=0.5, path="auto", workspace="auto"):
    Ws, cs = fn.fold_weights(T(Wt, dtype), T(g, "f32"), T(b, "f32"), T(c, "f32"))
    z = fn.linear(T(a, dtype), Ws, cs, eps=eps, mode=mode, alpha=alpha, path=path, workspace=workspace)
    torch.cuda.synchronize()
    return H(z)


@pytest.mark.parametrize("mode", ["rmsnorm", "layernorm", "dyt", "none"])
@pytest.mark.parametrize("eps", [1e-5, 0.0])
@pytest.mark.parametrize("bias", [False, True])
def test_f32_tiny_config(mode, eps, bias):
    """BASELINE config 1: 8 tokens, n=64 -> 64 outputs, fp32, <= 1e-5."""
    a, Wt, g, b, c, ref = _layer_and_ref(1, 8, 64, 64, "f32", mode, eps=eps, bias=bias, tiny=True)
    z = _run(a, Wt, g, b, c, "f32", mode, eps=eps)
    assert O.rowwise_rel_err(z, ref) <= TOL_F32


@pytest.mark.parametrize("M,K,N", [(3, 4096, 72), (33, 520, 8)])
@pytest.mark.parametrize("mode", ["rmsnorm", "dyt"])
def test_f32_larger(M, K, N, mode):
    a, Wt, g, b, c, ref = _layer_and_ref(2, M, K, N, "f32", mode)
    assert O.rowwise_rel_err(_run(a, Wt, g, b, c, "f32", mode), ref) <= TOL_F32


# ============================================================ linear: bf16 tcgen05 GEMM

GEMM_SHAPES = [(128, 64, 256), (300, 1000, 520), (17, 4096, 256), (1000, 4096, 1024), (257, 8192, 264)]


@pytest.mark.parametrize("M,K,N", GEMM_SHAPES)
@pytest.mark.parametrize("mode", ["rmsnorm", "layernorm", "dyt", "none"])
@pytest.mark.parametrize("path", ["gemm", "gemm1"])
def test_gemm_parity(M, K, N, mode, path):
    """path gemm: CTA-pair cta_group::2 kernel (M > 128, not DyT); gemm1: the 1-CTA kernel."""
    a, Wt, g, b, c, ref = _layer_and_ref(3, M, K, N, "bf16", mode)
    z = _run(a, Wt, g, b, c, "bf16", mode, path=path)
    err = O.rowwise_rel_err(z, ref)
    assert err <= TOL_BF16, err


@pytest.mark.parametrize("M,K,N", GEMM_SHAPES)
@pytest.mark.parametrize("path", ["gemm", "gemm1"])
def test_dyt_prologue_and_prepass(M, K, N, path):
    """DyT two ways: tanh in the A-tile prologue (workspace=None) and the K8 pre-pass into a
    workspace followed by the NONE GEMM.  Both meet the oracle; z is bit-identical (same bf16
    multiply + tanh.approx.bf16x2, include/flashnorm.h flashnorm_linear_ws)."""
    a, Wt, g, b, c, ref = _layer_and_ref(3, M, K, N, "bf16", "dyt")
    Ws, cs = fn.fold_weights(T(Wt), T(g, "f32"), T(b, "f32"), T(c, "f32"))
    ad = T(a)
    nb = fn.linear_workspace_bytes(M, K, N, "dyt", torch.bfloat16, path)
    assert nb >= 4096 + M * K * 2
    z_pro = fn.linear(ad, Ws, cs, mode="dyt", alpha=0.5, path=path, workspace=None)
    ws = torch.full((nb + 64,), 0x7F, dtype=torch.uint8, device=DEV)   # poisoned past the 4 KiB of flags, oversized
    ws[:4096] = 0
    n0 = fn.launch_count()
    z_pre = fn.linear(ad, Ws, cs, mode="dyt", alpha=0.5, path=path, workspace=ws)
    assert fn.launch_count() - n0 == 2
    assert O.rowwise_rel_err(H(z_pro), ref) <= TOL_BF16
    assert O.rowwise_rel_err(H(z_pre), ref) <= TOL_BF16
    assert torch.equal(z_pro, z_pre)


def test_linear_workspace_rules():
    M, K, N = 256, 128, 256
    a = SD.activations(9, M, K, DEV, torch.bfloat16)
    Wt = SD.layer(9, N, K, DEV, torch.bfloat16)[0]
    assert fn.linear_workspace_bytes(M, K, N, "rmsnorm", torch.bfloat16) == 0      # 2 pair tiles: no stream-K
    assert fn.linear_workspace_bytes(8, K, N, "dyt", torch.bfloat16) == 0          # decode GEMV
    assert fn.linear_workspace_bytes(8, K, N, "dyt", torch.bfloat16, "gemm1") == 4096 + 8 * K * 2
    assert fn.linear_workspace_bytes(M, K, N, "dyt", torch.float32) == 0
    # stream-K policy (FN_GEMM2_SK, read per call): off by default (measured no faster), 1 = the
    # mode-none kernel, 2 = also RMS; config 4 (128 pair tiles on 74 pairs) then needs its scratch
    assert fn.linear_workspace_bytes(2048, 4096, 4096, "none", torch.bfloat16) == 0
    os.environ["FN_GEMM2_SK"] = "1"
    try:
        assert fn.linear_workspace_bytes(2048, 4096, 4096, "none", torch.bfloat16) > 0
        assert fn.linear_workspace_bytes(2048, 4096, 4096, "rmsnorm", torch.bfloat16) == 0
        os.environ["FN_GEMM2_SK"] = "2"
        assert fn.linear_workspace_bytes(2048, 4096, 4096, "rmsnorm", torch.bfloat16) > 0
    finally:
        del os.environ["FN_GEMM2_SK"]
    small = torch.empty(4096 + M * K * 2 - 16, dtype=torch.uint8, device=DEV)
    with pytest.raises(fn.FlashNormError, match="workspace_bytes"):
        fn.linear(a, Wt, mode="dyt", workspace=small)
    z = torch.empty(M, N, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(fn.FlashNormError, match="alias"):
        fn.linear(a, Wt, mode="dyt", out=z, workspace=z)
    # non-DyT modes ignore a workspace
    ws = torch.empty(M * K * 2, dtype=torch.uint8, device=DEV)
    assert torch.equal(fn.linear(a, Wt, mode="rmsnorm", workspace=ws), fn.linear(a, Wt, mode="rmsnorm"))


@pytest.mark.parametrize("amode", ["outlier", "lowenergy"])
@pytest.mark.parametrize("eps", [1e-5, 0.0])
def test_gemm_input_modes(amode, eps):
    """Llama-style outlier channels and low-energy rows (which pin eps inside the sqrt, App. A)."""
    a, Wt, g, b, c, ref = _layer_and_ref(4, 384, 2048, 512, "bf16", "rmsnorm", amode=amode, eps=eps)
    z = _run(a, Wt, g, b, c, "bf16", "rmsnorm", eps=eps, path="gemm")
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16


def test_gemm_eps_placement_detectable():
    """A kernel with eps outside the sqrt would fail: low-energy rows make the readings differ."""
    a, Wt, g, b, c, ref = _layer_and_ref(5, 256, 1024, 256, "bf16", "rmsnorm", amode="lowenergy")
    z = _run(a, Wt, g, b, c, "bf16", "rmsnorm", path="gemm")
    r = O.rms(a)
    wrong = O.linear(a / (r + 1e-5)[:, None] * g + b, Wt.T, c)
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16 < O.rowwise_rel_err(wrong, ref)


# ============================================================ linear: bf16 decode GEMV

@pytest.mark.parametrize("M", [1, 5, 16])
@pytest.mark.parametrize("K,N", [(4096, 6144), (1000, 24), (8192, 136), (64, 8), (4160, 20000), (2048, 4104), (512, 40000),
                                 (520, 75776)])
@pytest.mark.parametrize("mode", ["rmsnorm", "dyt", "none"])
@pytest.mark.parametrize("path", ["gemv", "gemv_mma"])
def test_gemv_parity(M, K, N, mode, path):
    """gemv: tcgen05 split-K decode kernel (clusters of up to 8 CTAs; N=20000 has more 128-row tiles
    than SMs and runs 256-row tiles, N=40000 512-row tiles); gemv_mma: the mma.sync decode kernel."""
    if path == "gemv_mma" and M * K * 2 > 150 * 1024:
        path = "auto"
    a, Wt, g, b, c, ref = _layer_and_ref(6, M, K, N, "bf16", mode)
    z = _run(a, Wt, g, b, c, "bf16", mode, path=path)
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16


@pytest.mark.parametrize("M,K,N", [(1, 4096, 6144), (16, 4096, 6144), (3, 8192, 1024)])
@pytest.mark.parametrize("mode", ["rmsnorm", "dyt"])
def test_gemv_repeated_launches_bit_identical(M, K, N, mode):
    """split-K partials are summed in fixed rank order: every launch gives the same bits"""
    a = SD.activations(41, M, K, DEV, torch.bfloat16)
    Wt = SD.layer(41, N, K, DEV, torch.bfloat16)[0]
    z0 = fn.linear(a, Wt, mode=mode, path="gemv")
    for _ in range(5):
        assert torch.equal(fn.linear(a, Wt, mode=mode, path="gemv"), z0)


@pytest.mark.parametrize("M,K,N", [(17, 4096, 6144), (32, 4096, 6144), (48, 512, 1000), (64, 4096, 6144),
                                   (100, 1024, 2048), (128, 4096, 6144), (24, 8192, 1536)])
@pytest.mark.parametrize("mode", ["rmsnorm", "none", "layernorm", "dyt"])
def test_batched_decode_parity(M, K, N, mode):
    """17 <= M <= 128 (K4w, gemv_wide.cu): swap-AB tcgen05 with the tokens as the MMA N, split-K over a
    cluster with the peers' partials pushed to the leader — every output against the fp64 oracle,
    repeated launches bit-identical."""
    a, Wt, g, b, c, ref = _layer_and_ref(21, M, K, N, "bf16", mode)
    Ws, cs = fn.fold_weights(T(Wt, "bf16"), T(g, "f32"), T(b, "f32"), T(c, "f32"))
    at = T(a, "bf16")
    z = fn.linear(at, Ws, cs, mode=mode, eps=1e-5)
    z2 = fn.linear(at, Ws, cs, mode=mode, eps=1e-5)
    torch.cuda.synchronize()
    assert torch.equal(z, z2)
    assert O.rowwise_rel_err(z.float().cpu().numpy(), ref) <= TOL_BF16


@pytest.mark.parametrize("M", [17, 48, 128])
def test_batched_decode_linear_scaled(M):
    """The GLU / ReLU FFN down projection at 17..128 tokens (K4w, mode none with the per-row scale)
    against the oracle, and against the GEMM kernel (path='gemm1') within tolerance."""
    K, N = 2048, 4096
    a = gen_activations(22, M, K, "normal", "bf16")
    Wt, _, _, c = gen_layer(22, N, K, "bf16", with_c=True)
    s = np.linspace(0.25, 4.0, M).astype(np.float32)
    z = fn.linear_scaled(T(a, "bf16"), T(Wt, "bf16"), T(s, "f32"), c_star=T(c, "f32"))
    torch.cuda.synchronize()
    ref = O.linear(a, Wt.T) * s[:, None] + c[None, :]
    assert O.rowwise_rel_err(z.float().cpu().numpy(), ref) <= TOL_BF16


def test_decode_and_prefill_paths_agree():
    a, Wt, g, b, c, ref = _layer_and_ref(7, 16, 4096, 1024, "bf16", "rmsnorm")
    z1 = _run(a, Wt, g, b, c, "bf16", "rmsnorm", path="gemv")
    z2 = _run(a, Wt, g, b, c, "bf16", "rmsnorm", path="gemm")
    assert O.rowwise_rel_err(z1, ref) <= TOL_BF16 and O.rowwise_rel_err(z2, ref) <= TOL_BF16
    assert O.rowwise_rel_err(z1, z2) <= 1e-2


# ============================================================ edge cases

def test_empty_batch_is_noop():
    W = torch.zeros(64, 64, dtype=torch.bfloat16, device=DEV)
    z = fn.linear(torch.zeros(0, 64, dtype=torch.bfloat16, device=DEV), W)
    assert z.shape == (0, 64)


def test_zero_row_with_eps_zero_is_isolated():
    """A zero-energy row with eps=0 is IEEE inf/NaN in that row only (documented in flashnorm.h)."""
    a, Wt, g, b, c, ref = _layer_and_ref(8, 130, 512, 256, "bf16", "rmsnorm", bias=False)
    a[5] = 0.0
    for path in ("gemm", "gemv"):
        aa = a[:16].copy() if path == "gemv" else a
        z = _run(aa, Wt, g, None, None, "bf16", "rmsnorm", eps=0.0, path=path)
        assert not np.isfinite(z[5]).any()
        keep = [i for i in range(aa.shape[0]) if i != 5]
        assert O.rowwise_rel_err(z[keep], ref[: aa.shape[0]][keep]) <= TOL_BF16


def test_minimum_shapes():
    for M, K, N in [(1, 8, 8), (2, 8, 8), (129, 8, 8)]:
        a, Wt, g, b, c, ref = _layer_and_ref(9, M, K, N, "bf16", "rmsnorm")
        assert O.rowwise_rel_err(_run(a, Wt, g, b, c, "bf16", "rmsnorm"), ref) <= TOL_BF16


def test_alignment_error_raised():
    w = torch.zeros(64, 64, dtype=torch.bfloat16, device=DEV)
    a = torch.zeros(4 * 64 + 1, dtype=torch.bfloat16, device=DEV)[1:].view(4, 64)
    with pytest.raises(fn.FlashNormError, match="FN_ERR_ALIGN"):
        fn.linear(a, w)


# ============================================================ config 4: LayerNorm retrofit + DyT

def test_config4_layernorm_retrofit_end_to_end():
    """x -> V* (mean centering folded) -> FlashNorm linear (LN g,b folded)."""
    M, d = 2048, 4096
    x, Vt, bp = gen_upstream(21, M, d, d, "bf16")
    Wt, g, b, c = gen_layer(21, d, d, "bf16", with_b=True, with_c=True)
    Vs, bs = fn.fold_mean_center(T(Vt), T(bp, "f32"))
    a_star = fn.linear(T(x), Vs, bs, mode="none")            # upstream layer, outputs centered
    Ws, cs = fn.fold_weights(T(Wt), T(g, "f32"), T(b, "f32"), T(c, "f32"))
    z = H(fn.linear(a_star, Ws, cs, eps=1e-5, mode="layernorm"))
    rows = np.r_[0, 1, M - 1, np.random.default_rng(0).choice(M, 29, replace=False)]
    ref = O.upstream_layernorm_linear(x[rows], Vt.T, bp, Wt.T, g, b, c, 1e-5)
    assert O.rowwise_rel_err(z[rows], ref) <= TOL_BF16


def test_config4_dyt_variant():
    M, d = 2048, 4096
    a = gen_activations(22, M, d, "normal", "bf16")
    Wt, g, b, c = gen_layer(22, d, d, "bf16", with_b=True, with_c=True)
    z = _run(a, Wt, g, b, c, "bf16", "dyt", alpha=0.5)
    rows = np.r_[0, M - 1, np.random.default_rng(1).choice(M, 30, replace=False)]
    ref = O.norm_linear(a[rows], Wt.T, g, b, c, 0.0, "dyt", 0.5)
    assert O.rowwise_rel_err(z[rows], ref) <= TOL_BF16


# ============================================================ full BASELINE sizes (bench launch config)

def _oracle_rows(a_rows, Wt_dev, g, b, c, eps, mode, alpha=0.5, col_chunk=4096):
    """Oracle on sampled rows, W streamed to the host in column chunks (memory only)."""
    N = Wt_dev.shape[0]
    out = np.empty((a_rows.shape[0], N))
    for j0 in range(0, N, col_chunk):
        j1 = min(N, j0 + col_chunk)
        W = Wt_dev[j0:j1].float().cpu().numpy().T
        out[:, j0:j1] = O.norm_linear(a_rows, W, g, b, None if c is None else c[j0:j1], eps, mode, alpha)
    return out


def _rows_per_block(M, per_block, seed, extra=(), block=256):
    """per_block seeded rows from every `block`-row M block (the pair kernel's 256-row tiles),
    plus the fixed `extra` rows (first/last rows, tile edges)."""
    rng = np.random.default_rng(seed)
    rows = set(int(r) for r in extra)
    for m0 in range(0, M, block):
        m1 = min(M, m0 + block)
        rows.update(int(r) for r in rng.choice(np.arange(m0, m1), min(per_block, m1 - m0), replace=False))
    return np.array(sorted(rows))


def _full_size(M, K, N, seed, mode="rmsnorm", with_bias=False):
    a = SD.activations(seed, M, K, DEV, torch.bfloat16)
    Wt, g, b, c = SD.layer(seed, N, K, DEV, torch.bfloat16, with_b=with_bias, with_c=with_bias)
    Ws, cs = fn.fold_weights(Wt, g, b, c)
    return a, Wt, g, b, c, Ws, cs


@pytest.mark.parametrize("M", [1, 16])
def test_config2_decode_full(M):
    """Llama-3-8B decode: RMSNorm + QKV 4096 -> 6144, all outputs vs oracle."""
    a, Wt, g, b, c, Ws, cs = _full_size(M, 4096, 6144, 31)
    z = H(fn.linear(a, Ws, cs, eps=1e-5))
    ref = _oracle_rows(H(a), Wt, H(g), None, None, 1e-5, "rmsnorm")
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16


@pytest.mark.parametrize("M", [1, 16])
def test_decode_wide_n_70b_gate_up(M):
    """Decode through the tcgen05 kernel for N > 256 x #SMs: the Llama-3-70B gate||up shape (K = 8192,
    N = 57344 = 112 tiles of 512 rows), every output against the fp64 oracle."""
    a, Wt, g, b, c, Ws, cs = _full_size(M, 8192, 57344, 34)
    n0 = fn.launch_count()
    z = H(fn.linear(a, Ws, cs, eps=1e-5, path="gemv"))
    assert fn.launch_count() - n0 == 1
    ref = _oracle_rows(H(a), Wt, H(g), None, None, 1e-5, "rmsnorm")
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16


def test_config3_prefill_full_sampled():
    """Llama-3-8B prefill: 4096 tokens, 4096 -> 28672 (gate||up), exactly as bench.py launches it."""
    M, K, N = 4096, 4096, 28672
    a, Wt, g, b, c, Ws, cs = _full_size(M, K, N, 32)
    z = fn.linear(a, Ws, cs, eps=1e-5)
    z2 = fn.linear(a, Ws, cs, eps=1e-5)
    torch.cuda.synchronize()
    assert torch.equal(z, z2), "not deterministic"
    rows = _rows_per_block(M, 2, seed=2, extra=(0, 1, 127, 128, M - 1))
    assert len({r // 256 for r in rows}) == M // 256            # every 256-row M block of the pair kernel
    ref = _oracle_rows(H(a[torch.as_tensor(rows, device=DEV)]), Wt, H(g), None, None, 1e-5, "rmsnorm")
    assert O.rowwise_rel_err(H(z)[rows], ref) <= TOL_BF16
    # row-permutation equivariance (rows are independent): bit-exact
    perm = torch.randperm(M, generator=torch.Generator().manual_seed(3)).to(DEV)
    zp = fn.linear(a[perm].contiguous(), Ws, cs, eps=1e-5)
    torch.cuda.synchronize()
    assert torch.equal(zp, z[perm])


@pytest.mark.slow
def test_config5_column_shards_concatenate_bit_exact():
    """Llama-3-70B FFN shapes, W* column-sharded P = 8 ways: the concatenated shards are
    bit-identical to the unsharded result (per-tile math is independent of P)."""
    M, K, N, P = 8192, 8192, 57344, 8
    a, Wt, g, b, c, Ws, cs = _full_size(M, K, N, 33)
    z = fn.linear(a, Ws, cs, eps=1e-5)
    Nl = N // P
    for p in range(P):
        zp = fn.linear(a, Ws[p * Nl:(p + 1) * Nl], None, eps=1e-5)
        assert torch.equal(zp, z[:, p * Nl:(p + 1) * Nl]), p
        del zp
    del Ws
    # 2 rows from every one of the 32 M blocks (64 rows), against the UNFUSED oracle built from
    # the original W and g (RMSNorm then the linear layer, Fig 1(a)) -- not from the GPU fold
    rows = _rows_per_block(M, 2, seed=4)
    assert len(rows) == 64 and len({r // 256 for r in rows}) == M // 256
    zr = H(z[torch.as_tensor(rows, device=DEV)])
    del z
    ref = _oracle_rows(H(a[torch.as_tensor(rows, device=DEV)]), Wt, H(g), None, None, 1e-5, "rmsnorm")
    assert O.rowwise_rel_err(zr, ref) <= TOL_BF16


def test_baseline_unfused_matches_oracle():
    """The measurement-only unfused variant (RMSNorm kernel -> plain GEMM on the original W)."""
    a, Wt, g, b, c, ref = _layer_and_ref(10, 512, 2048, 768, "bf16", "rmsnorm")
    y = fn.baseline_norm(T(a), T(g, "f32"), T(b, "f32"), eps=1e-5)
    z = H(fn.linear(y, T(Wt), T(c, "f32"), mode="none"))
    assert O.rowwise_rel_err(z, ref) <= TOL_BF16


def test_gather_columns_permute():
    P, M, Nl = 4, 37, 64
    parts = torch.randn(P, M, Nl, device=DEV).to(torch.bfloat16)
    z = fn.gather_columns(parts)
    torch.cuda.synchronize()
    assert torch.equal(z, parts.permute(1, 0, 2).reshape(M, P * Nl))


@pytest.mark.parametrize("M,K,N", [(4096, 512, 28672), (256, 512, 28672), (2048, 64, 8192), (9000, 256, 4096)])
@pytest.mark.parametrize("mode", ["rmsnorm", "dyt", "none"])
@pytest.mark.parametrize("path", ["gemm", "gemm1"])
def test_gemm_repeated_launches_bit_identical(M, K, N, mode, path):
    """(9000, 256, 4096): 36 pair M blocks > the 16-slot ssq cache -> slot replacement; ragged M."""
    """Regression for the stage-release race (ssq group vs TMA refill): many tiles per CTA,
    W* streamed from HBM; every launch must produce identical bits."""
    a = SD.activations(40, M, K, DEV, torch.bfloat16)
    Wt, g, b, c = SD.layer(40, N, K, DEV, torch.bfloat16, with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(Wt, g, b, c)
    z0 = fn.linear(a, Ws, cs, eps=1e-5, mode=mode, path=path)
    for _ in range(5):
        assert torch.equal(fn.linear(a, Ws, cs, eps=1e-5, mode=mode, path=path), z0)
    # against the unfused fp64 oracle (original W, g, b, c) on rows from every 256-row M block
    # ((9000, 256, 4096): 36 blocks, so cached slots are replaced and revisited)
    rows = _rows_per_block(M, 2, seed=M + K, extra=(M - 1,))
    ah = H(a[torch.as_tensor(rows, device=DEV)])
    if mode == "none":
        ref = O.linear(ah, H(Ws).T, H(cs))
    else:
        ref = O.norm_linear(ah, H(Wt).T, H(g), H(b), H(c), 1e-5, mode, 0.5)
    assert O.rowwise_rel_err(H(z0)[rows], ref) <= TOL_BF16


# ============================================================ NEXT-3: column gather fused into the epilogue

@pytest.mark.parametrize("M", [4, 77, 300])
@pytest.mark.parametrize("mode", ["rmsnorm", "none", "dyt"])
def test_linear_gather_shards_into_every_destination_bit_exact(M, mode):
    """Each of P = 4 column shards writes itself (flashnorm_linear_gather) into ndst = 3 [M x N]
    buffers; afterwards every buffer equals the unsharded flashnorm_linear bit for bit (the
    shard-concatenation invariant of SURVEY §8(e), through the multi-destination epilogue)."""
    K, N, P = 512, 1024, 4
    a = T(gen_activations(61, M, K, "normal", "bf16"))
    Wt, g, b, c = gen_layer(61, N, K, "bf16", with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(T(Wt), T(g, "f32"), T(b, "f32"), T(c, "f32"))
    full = fn.linear(a, Ws, cs, eps=1e-5, mode=mode, alpha=0.5, path="gemm")
    dsts = [torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=DEV) for _ in range(3)]
    Nl = N // P
    for r in range(P):
        fn.linear_gather(a, Ws[r * Nl:(r + 1) * Nl], dsts, r * Nl, c_star=cs[r * Nl:(r + 1) * Nl], eps=1e-5,
                         mode=mode, alpha=0.5)
    for d in dsts:
        assert np.array_equal(bits(d), bits(full))


def test_linear_gather_strided_destination_and_validation():
    """A shard into a wider row (ldz > N, col0 > 0) leaves the other columns untouched; bad
    arguments are rejected before any launch."""
    M, K, N, ldz, col0 = 130, 256, 256, 1024, 512
    a = T(gen_activations(62, M, K, "normal", "bf16"))
    Wt, g, _, _ = gen_layer(62, N, K, "bf16")
    Ws, cs = fn.fold_weights(T(Wt), T(g, "f32"))
    z = fn.linear(a, Ws, cs, eps=1e-5)
    dst = torch.zeros((M, ldz), dtype=torch.bfloat16, device=DEV)
    fn.linear_gather(a, Ws, [dst], col0, c_star=cs)
    assert np.array_equal(bits(dst[:, col0:col0 + N].contiguous()), bits(z))
    assert not dst[:, :col0].any() and not dst[:, col0 + N:].any()
    with pytest.raises(fn.FlashNormError, match="FN_ERR_SHAPE"):
        fn.linear_gather(a, Ws, [dst], ldz - N + 8, c_star=cs)
    with pytest.raises(fn.FlashNormError, match="FN_ERR_VALUE"):
        fn.linear_gather(a, Ws, [dst] * 9, 0, c_star=cs)


@pytest.mark.parametrize("M", [8, 300, 2500])
def test_linear_from_host_matches_device_path(M):
    """The end-to-end entry (pinned host buffers; M >= 1024 pipelined in row chunks over copy
    streams) returns exactly the device path's z, also when called back to back."""
    K, N = 512, 1024
    a = T(gen_activations(71, M, K, "normal", "bf16"))
    Wt, g, b, c = gen_layer(71, N, K, "bf16", with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(T(Wt), T(g, "f32"), T(b, "f32"), T(c, "f32"))
    ref = bits(fn.linear(a, Ws, cs, eps=1e-5))
    a_host = a.cpu().pin_memory()
    z_host = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
    a_dev, z_dev = torch.empty_like(a), torch.empty((M, N), dtype=torch.bfloat16, device=DEV)
    for _ in range(3):
        z_host.zero_()
        fn.linear_from_host(a_host, Ws, cs, a_dev, z_dev, z_host)
        torch.cuda.current_stream().synchronize()
        assert np.array_equal(z_host.view(torch.int16).numpy().view(np.uint16), ref)


_DEBUG_LN = r'''
import sys
sys.path.insert(0, sys.argv[1])
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
a = SD.activations(5, 64, 512, "cuda", torch.bfloat16)
W = SD.layer(5, 256, 512, "cuda", torch.bfloat16)[0]
ac = (a.float() - a.float().mean(1, keepdim=True)).to(torch.bfloat16)   # mean-centered rows
fn.linear(ac, W, mode="layernorm")
try:
    fn.linear(a + 1.0, W, mode="layernorm")                             # |mean|/rms ~ 0.7
    print("NOT_REJECTED")
except fn.FlashNormError as e:
    print("REJECTED" if "not mean-centered" in str(e) else "OTHER " + str(e))
'''


def test_layernorm_debug_check_rejects_uncentered_input():
    """include/flashnorm.h FN_LAYERNORM: with FN_DEBUG_LAYERNORM=1 an input that was not
    mean-centered upstream is reported as FN_ERR_VALUE; a centered one passes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _DEBUG_LN, root], env=dict(os.environ, FN_DEBUG_LAYERNORM="1"),
                       capture_output=True, text=True, timeout=300)
    assert "REJECTED" in r.stdout and "NOT_REJECTED" not in r.stdout, r.stdout + r.stderr[-3000:]


def test_linear_gather_multicast_validation():
    """flashnorm_linear_gather_multicast rejects bad arguments before any launch (the store path
    itself needs an NVLS multicast mapping: tests/test_gpu_multi.py on a multi-GPU NVSwitch node)."""
    M, K, N = 64, 256, 256
    a = T(gen_activations(63, M, K, "normal", "bf16"))
    Wt, g, _, _ = gen_layer(63, N, K, "bf16")
    Ws, cs = fn.fold_weights(T(Wt), T(g, "f32"))
    with pytest.raises(fn.FlashNormError, match="FN_ERR_NULL"):
        fn.linear_gather_multicast(a, Ws, 0, N, 0, c_star=cs)
    with pytest.raises(fn.FlashNormError, match="FN_ERR_SHAPE"):
        fn.linear_gather_multicast(a, Ws, 1 << 40, N - 8, 0, c_star=cs)
    with pytest.raises(fn.FlashNormError, match="FN_ERR_ALIGN"):
        fn.linear_gather_multicast(a, Ws, (1 << 40) + 8, N, 0, c_star=cs)


# ============================================================ stream-K tail of the pair kernel

@pytest.mark.parametrize("M,K,N,mode", [(2048, 4096, 4096, "rmsnorm"), (2048, 4096, 4096, "none"),
                                        (2048, 4096, 4096, "layernorm"), (2048, 4096, 4096, "dyt"),
                                        (4096, 1024, 2816, "rmsnorm"), (2304, 520, 4104, "rmsnorm"),
                                        (2048, 192, 4096, "rmsnorm")])
def test_stream_k_tail_parity_and_determinism(M, K, N, mode, monkeypatch):
    """Shapes whose pair-tile count is not a multiple of the 74 CTA pairs (config 4: 128 tiles) run
    the stream-K tail when a workspace is given: every 256-row M block against the fp64 oracle, and
    repeated calls (flags reset, partial order fixed) bit-identical; the no-workspace (whole-tile)
    result agrees within the tolerance.  FN_GEMM2_SK=2 (read per call) extends the tail to the RMS
    kernel, which the default policy keeps whole-tile."""
    monkeypatch.setenv("FN_GEMM2_SK", "2")
    a, Wt, g, b, c, ref = _layer_and_ref(81, M, K, N, "bf16", mode)
    Ws, cs = fn.fold_weights(T(Wt), T(g, "f32"), T(b, "f32"), T(c, "f32"))
    at = T(a)
    nb = fn.linear_workspace_bytes(M, K, N, mode, torch.bfloat16)
    assert nb > 0
    ws = torch.zeros(nb, dtype=torch.uint8, device=DEV)
    z0 = fn.linear(at, Ws, cs, eps=1e-5, mode=mode, alpha=0.5, workspace=ws)
    for _ in range(3):
        assert torch.equal(fn.linear(at, Ws, cs, eps=1e-5, mode=mode, alpha=0.5, workspace=ws), z0)
    assert not ws[:4096].any(), "stream-K flags not left zero"
    assert O.rowwise_rel_err(H(z0), ref) <= TOL_BF16
    z_whole = fn.linear(at, Ws, cs, eps=1e-5, mode=mode, alpha=0.5, workspace=None if mode != "dyt" else "auto")
    assert O.rowwise_rel_err(H(z_whole), ref) <= TOL_BF16


def test_stream_k_tail_graph_replay(monkeypatch):
    """The stream-K flags end every call at zero, so a captured CUDA graph replays correctly with a
    changing input."""
    monkeypatch.setenv("FN_GEMM2_SK", "2")
    M, K, N = 2048, 1024, 4096
    a0 = gen_activations(82, M, K, "normal", "bf16")
    a1 = gen_activations(83, M, K, "normal", "bf16")
    Wt, g, _, _ = gen_layer(82, N, K, "bf16")
    Ws, _ = fn.fold_weights(T(Wt), T(g, "f32"))
    nb = fn.linear_workspace_bytes(M, K, N, "rmsnorm", torch.bfloat16)
    ws = torch.zeros(nb, dtype=torch.uint8, device=DEV)
    ain = T(a0)
    z = torch.empty((M, N), dtype=torch.bfloat16, device=DEV)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn.linear(ain, Ws, None, out=z, workspace=ws)
        st.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            fn.linear(ain, Ws, None, out=z, workspace=ws)
    for a in (a1, a0, a1):
        ain.copy_(T(a))
        gr.replay()
        torch.cuda.synchronize()
        ref = O.norm_linear(a, Wt.T, g, None, None, 1e-5, "rmsnorm")
        assert O.rowwise_rel_err(H(z), ref) <= TOL_BF16
