"""Pins for the fp64 oracle (oracle/flashnorm_oracle.py) — CPU only.

The oracle is pinned to things other than itself:
  * hand-derived worked examples with citations (tests/golden/worked_examples.json),
  * closed forms and the paper's identities,
  * an independent library routine (torch.nn.functional.rms_norm / layer_norm in
    float64, math.tanh) on random inputs,
  * brute force with exact rational arithmetic (fractions) on tiny inputs,
  * fault injection: plausible mistakes (eps outside sqrt, 1/(n-1), bias before
    scale, c* from W*, dropped b_prev centering) must FAIL at least one pin.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import flashnorm_oracle as O


def ev(expr):
    return float(eval(str(expr), {"__builtins__": {}}, {k: getattr(math, k) for k in ("sqrt", "tanh", "exp")}))


def evv(lst):
    return np.array([ev(e) for e in lst], dtype=np.float64)


# ---------------------------------------------------------------- worked examples

def test_rms_family_worked(golden):
    for ex in golden["rms"]:
        assert O.rms(np.array(ex["a"], float)) == pytest.approx(ev(ex["expect"]), rel=1e-15, abs=0), ex["cite"]
    for ex in golden["rmse"]:
        assert O.rmse(np.array(ex["a"], float), ex["eps"]) == pytest.approx(ev(ex["expect"]), rel=1e-15), ex["cite"]
    for ex in golden["rss"]:
        assert O.rss(np.array(ex["a"], float)) == pytest.approx(ev(ex["expect"]), rel=1e-15), ex["cite"]
    for ex in golden["rsse"]:
        assert O.rsse(np.array(ex["a"], float), ex["eps"]) == pytest.approx(ev(ex["expect"]), rel=1e-15), ex["cite"]


def test_mean_center_worked(golden):
    for ex in golden["mean_center"]:
        np.testing.assert_allclose(O.mean_center(np.array(ex["y"], float)), evv(ex["expect"]), atol=1e-15)


def test_norms_worked(golden):
    for ex in golden["norms"]:
        y = O.normalize(np.array(ex["a"], float), ex["mode"], ex["g"], ex["b"], ex["eps"],
                        ex["alpha"] if ex["alpha"] is not None else 0.5)
        np.testing.assert_allclose(y, evv(ex["expect"]), rtol=1e-14, atol=1e-15, err_msg=ex["cite"])


def test_norm_linear_worked(golden):
    for ex in golden["norm_linear"]:
        z = O.norm_linear(np.array(ex["a"], float), np.array(ex["W"], float), ex["g"], ex["b"], ex["c"],
                          ex["eps"], ex["mode"])
        np.testing.assert_allclose(z, np.array([evv(r) for r in ex["expect"]]), rtol=1e-14, err_msg=ex["cite"])


def test_folds_worked(golden):
    for ex in golden["fold_weights"]:
        Ws, cs = O.fold_weights(np.array(ex["W"], float), ex["g"], ex["b"], ex["c"])
        np.testing.assert_array_equal(Ws, np.array(ex["W_star"], float), err_msg=ex["cite"])
        if ex["c_star"] is not None:
            np.testing.assert_array_equal(cs, np.array(ex["c_star"], float), err_msg=ex["cite"])
    for ex in golden["fold_mean_center"]:
        V = np.array(ex["V"], float)
        np.testing.assert_array_equal(O.row_sums(V), np.array(ex["s"], float))
        Vs, bs = O.fold_mean_center(V, ex["b_prev"])
        np.testing.assert_array_equal(Vs, np.array(ex["V_star"], float), err_msg=ex["cite"])
        if ex["b_prev_star"] is not None:
            np.testing.assert_array_equal(bs, np.array(ex["b_prev_star"], float))


def test_mean_retrofit_worked(golden):
    for ex in golden["mean_retrofit"]:
        x, V = np.array(ex["x"], float), np.array(ex["V"], float)
        np.testing.assert_array_equal(O.linear(x, V), np.array(ex["y"], float))
        assert O.mean_via_s(x, V) == ev(ex["mu"])
        Vs, _ = O.fold_mean_center(V)
        np.testing.assert_allclose(O.linear(x, Vs), np.array(ex["centered"], float), atol=1e-15)


# ---------------------------------------------------------------- independent library routines

@pytest.mark.parametrize("eps", [0.0, 1e-5, 0.3])
def test_rmsnorm_matches_torch_f64(eps):
    import torch
    rng = np.random.default_rng(1)
    a = rng.standard_normal((7, 48)) * rng.uniform(0.01, 10, (7, 1))
    g = rng.uniform(0.5, 1.5, 48)
    ref = torch.nn.functional.rms_norm(torch.from_numpy(a), (48,), torch.from_numpy(g), eps=eps).numpy()
    np.testing.assert_allclose(O.rmsnorm(a, g, None, eps), ref, rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("eps", [0.0, 1e-5, 0.3])
def test_layernorm_matches_torch_f64(eps):
    import torch
    rng = np.random.default_rng(2)
    a = rng.standard_normal((5, 40)) * 3 + 7.0
    g = rng.uniform(0.5, 1.5, 40)
    b = rng.uniform(-0.1, 0.1, 40)
    ref = torch.nn.functional.layer_norm(torch.from_numpy(a), (40,), torch.from_numpy(g), torch.from_numpy(b),
                                         eps=eps).numpy()
    np.testing.assert_allclose(O.layernorm(a, g, b, eps), ref, rtol=1e-12, atol=1e-13)


def test_dyt_matches_math_tanh():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((3, 16)) * 4
    g = rng.uniform(0.5, 1.5, 16)
    b = rng.uniform(-0.1, 0.1, 16)
    ref = np.array([[g[k] * math.tanh(0.7 * a[m, k]) + b[k] for k in range(16)] for m in range(3)])
    np.testing.assert_allclose(O.dyt(a, g, b, 0.7), ref, rtol=1e-15, atol=1e-15)


def test_identity_weights_reduce_to_rmsnorm():
    """Special case W = I, g = 1, no biases: z = a / RMSe(a) (textbook RMSNorm)."""
    import torch
    rng = np.random.default_rng(4)
    a = rng.standard_normal((6, 32))
    z = O.norm_linear(a, np.eye(32), None, None, None, 1e-5, "rmsnorm")
    ref = torch.nn.functional.rms_norm(torch.from_numpy(a), (32,), eps=1e-5).numpy()
    np.testing.assert_allclose(z, ref, rtol=1e-13)


# ---------------------------------------------------------------- exact brute force (fractions)

def _brute_norm_linear_exact(a, W, g, b, c, mode, eps_num):
    """Exact rational evaluation of Fig 1(a) except for one sqrt (done last in float)."""
    M, n = len(a), len(a[0])
    k = len(W[0])
    out = []
    for m in range(M):
        x = [Fraction(v) for v in a[m]]
        if mode == "layernorm":
            mu = sum(x, Fraction(0)) / n
            x = [v - mu for v in x]
        ms = sum((v * v for v in x), Fraction(0)) / n + Fraction(eps_num)
        r = 1.0 / math.sqrt(ms)  # only irrational step
        # z_j = r * sum_i x_i g_i W_ij + sum_i b_i W_ij + c_j  (expanded exactly)
        row = []
        for j in range(k):
            lin = sum((x[i] * Fraction(g[i]) * Fraction(W[i][j]) for i in range(n)), Fraction(0))
            bias = sum((Fraction(b[i]) * Fraction(W[i][j]) for i in range(n)), Fraction(0)) + Fraction(c[j])
            row.append(float(lin) * r + float(bias))
        out.append(row)
    return np.array(out)


@pytest.mark.parametrize("mode", ["rmsnorm", "layernorm"])
def test_brute_force_tiny(mode):
    rng = np.random.default_rng(5)
    M, n, k = 3, 5, 4
    a = rng.integers(-9, 10, (M, n)) / 4.0
    W = rng.integers(-9, 10, (n, k)) / 8.0
    g = rng.integers(1, 9, n) / 4.0
    b = rng.integers(-4, 5, n) / 16.0
    c = rng.integers(-4, 5, k) / 16.0
    eps = 0.0625
    ref = _brute_norm_linear_exact(a.tolist(), W.tolist(), g, b, c, mode, eps)
    z = O.norm_linear(a, W, g, b, c, eps, mode)
    np.testing.assert_allclose(z, ref, rtol=1e-13, atol=1e-13)


# ---------------------------------------------------------------- the paper's identities (fp64, random)

def _rand_layer(seed, M=8, n=64, k=48):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((M, n))
    W = rng.standard_normal((n, k)) / np.sqrt(n)
    g = rng.uniform(0.5, 1.5, n)
    b = rng.uniform(-0.1, 0.1, n)
    c = rng.uniform(-0.1, 0.1, k)
    return a, W, g, b, c


@pytest.mark.parametrize("eps", [0.0, 1e-5])
def test_identity_merged_and_deferred(eps):
    """(a r g) W + ... = (a r) W* = (a W*) r, bias after scale."""
    a, W, g, b, c = _rand_layer(6)
    ref = O.norm_linear(a, W, g, b, c, eps, "rmsnorm")
    Ws, cs = O.fold_weights(W, g, b, c)
    merged = O.linear(O.rmsnorm(a, None, None, eps), Ws, cs)
    deferred = O.deferred_linear(a, Ws, cs, eps)
    assert O.rowwise_rel_err(merged, ref) < 1e-13
    assert O.rowwise_rel_err(deferred, ref) < 1e-13


def test_identity_bias_elimination():
    """(y + b) W + c = y W + (c + b W)."""
    a, W, g, b, c = _rand_layer(7)
    y = O.rmsnorm(a, g, None, 1e-5)
    lhs = O.linear(y + b, W, c)
    rhs = O.linear(y, W, O.eliminate_norm_bias(W, b, c))
    assert O.rowwise_rel_err(rhs, lhs) < 1e-13


def test_identity_mean_via_row_sums_and_vstar():
    """mu = x s / n = mean(x V) and x V* = mean_center(x V)."""
    rng = np.random.default_rng(8)
    x = rng.standard_normal((9, 24))
    V = rng.standard_normal((24, 40)) + rng.uniform(-0.5, 0.5, (24, 1))
    bp = rng.uniform(-0.5, 1.5, 40)
    np.testing.assert_allclose(O.mean_via_s(x, V), np.mean(x @ V, axis=1), rtol=1e-13)
    Vs, bs = O.fold_mean_center(V, bp)
    assert np.max(np.abs(Vs.sum(axis=1))) <= 1e-12 * 40
    np.testing.assert_allclose(O.linear(x, Vs, bs), O.mean_center(O.linear(x, V, bp)), atol=1e-12)


def test_identity_layernorm_retrofit():
    """LayerNorm after V  ==  RMSNorm after V* (PAPER.md:49 'retrofit ... without retraining')."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((6, 32))
    V = rng.standard_normal((32, 48)) / 6 + rng.uniform(-0.3, 0.3, (32, 1))
    bp = rng.uniform(-0.5, 1.5, 48)
    W = rng.standard_normal((48, 16)) / 7
    g, b, c = rng.uniform(0.5, 1.5, 48), rng.uniform(-0.1, 0.1, 48), rng.uniform(-0.1, 0.1, 16)
    ref = O.upstream_layernorm_linear(x, V, bp, W, g, b, c, 1e-5)
    Vs, bs = O.fold_mean_center(V, bp)
    Ws, cs = O.fold_weights(W, g, b, c)
    got = O.deferred_linear(O.linear(x, Vs, bs), Ws, cs, 1e-5)
    assert O.rowwise_rel_err(got, ref) < 1e-12


def test_identity_dyt_fold():
    """DyT bias/weights fold the same way: z = tanh(alpha a) W* + c*."""
    a, W, g, b, c = _rand_layer(10)
    ref = O.norm_linear(a, W, g, b, c, 0.0, "dyt", 0.5)
    Ws, cs = O.fold_weights(W, g, b, c)
    assert O.rowwise_rel_err(O.linear(np.tanh(0.5 * a), Ws, cs), ref) < 1e-13


def test_appendix_identities():
    """RMS = sqrt(1/n) RSS; RMSe = sqrt(1/n) RSSe; g* = sqrt(n) g gives the same y."""
    rng = np.random.default_rng(11)
    a = rng.standard_normal((5, 64))
    g = rng.uniform(0.5, 1.5, 64)
    np.testing.assert_allclose(O.rms(a), np.sqrt(1 / 64) * O.rss(a), rtol=1e-15)
    np.testing.assert_allclose(O.rmse(a, 1e-5), np.sqrt(1 / 64) * O.rsse(a, 1e-5), rtol=1e-15)
    np.testing.assert_allclose(O.rmsnorm(a, g, None, 0.0), a / O.rss(a)[:, None] * (np.sqrt(64) * g), rtol=1e-14)
    np.testing.assert_allclose(O.mean_square(a), O.rms(a) ** 2, rtol=1e-14)


def test_rms_scale_invariance():
    """RMS(s a) = s RMS(a), exact only without eps."""
    rng = np.random.default_rng(12)
    a = rng.standard_normal((4, 64))
    for s in (1e-3, 0.5, 7.0):
        np.testing.assert_allclose(O.rms(s * a), s * O.rms(a), rtol=1e-14)
        np.testing.assert_allclose(O.rmsnorm(s * a, None, None, 0.0), O.rmsnorm(a, None, None, 0.0), rtol=1e-13)
    # with eps the invariance breaks for low-energy vectors (App. A / PAPER.md:128)
    assert not np.allclose(O.rmsnorm(1e-3 * a, None, None, 1e-5), O.rmsnorm(a, None, None, 1e-5), rtol=1e-3)


# ---------------------------------------------------------------- fault injection: pins are not vacuous

def test_faults_are_detected(golden):
    ex = golden["rmse"][2]
    a = np.array(ex["a"], float)
    eps_outside = O.rms(a) + ex["eps"]                    # 1/(rms + eps) reading
    assert abs(eps_outside - ev(ex["expect"])) > 1e-6
    a34 = np.array([3.0, 4.0])
    unbiased = np.sqrt(np.sum(a34 ** 2) / (2 - 1))          # 1/(n-1)
    assert abs(unbiased - ev(golden["rms"][1]["expect"])) > 1e-3
    fw = golden["fold_weights"][2]
    W = np.array(fw["W"], float)
    Ws = O.merge_norm_weights(W, fw["g"])
    cs_wrong = np.array(fw["c"]) + np.array(fw["b"]) @ Ws   # c* built from W* (reading c5 violated)
    assert not np.allclose(cs_wrong, fw["c_star"])
    nl = golden["norm_linear"][0]
    a2, W2 = np.array(nl["a"], float), np.array(nl["W"], float)
    Ws2, cs2 = O.fold_weights(W2, nl["g"], nl["b"], nl["c"])
    bias_before_scale = (a2 @ Ws2 + cs2) / O.rms(a2)[:, None]  # reading c4 violated
    assert not np.allclose(bias_before_scale, [[ev(e) for e in nl["expect"][0]]], rtol=1e-3)
    fm = golden["fold_mean_center"][0]
    _, bs = O.fold_mean_center(np.array(fm["V"], float), None)
    assert bs is None  # dropping b_prev centering leaves b_prev un-centered: [1,3] != [-1,1]
    assert not np.allclose(fm["b_prev"], fm["b_prev_star"])


# ---------------------------------------------------------------- GLU FFN (NEXT-1)

def test_glu_worked(golden):
    for ex in golden["glu"]:
        a, g = np.array(ex["a"], float), np.array(ex["g"], float)
        Wg, Wu, Wd = (np.array(ex[k], float) for k in ("Wg", "Wu", "Wd"))
        h = O.glu_hidden(a, Wg, Wu, g, ex["eps"], ex["act"])
        np.testing.assert_allclose(h[0], evv(ex["expect_h"]), rtol=1e-14, atol=1e-15)
        if "expect_y" in ex:
            np.testing.assert_allclose(O.glu_ffn(a, Wg, Wu, Wd, g, ex["eps"], ex["act"])[0], evv(ex["expect_y"]),
                                       rtol=1e-14, atol=1e-15)
        Wgs, Wus = O.merge_norm_weights(Wg, g), O.merge_norm_weights(Wu, g)
        _, s = O.glu_hidden_deferred(a, Wgs, Wus, ex["eps"], ex["act"])
        assert s[0] == pytest.approx(ev(ex["expect_s_deferred"]), rel=1e-14)


def test_glu_act_textbook():
    """silu against math.exp per element; relu/bilinear against their definitions"""
    xs = np.linspace(-30, 30, 121)
    np.testing.assert_allclose(O.glu_act(xs, "silu"), [x / (1 + math.exp(-x)) for x in xs], rtol=1e-15, atol=1e-300)
    assert np.array_equal(O.glu_act(xs, "relu"), [max(x, 0.0) for x in xs])
    assert np.array_equal(O.glu_act(xs, "bilinear"), xs)


def _brute_glu_exact(a, Wg, Wu, Wd, g, eps, act):
    """Fractions for every step except the one irrational value, 1/RMSe (sqrt)."""
    out = []
    for row in a:
        n = len(row)
        ms = sum(Fraction(x) ** 2 for x in row) / n + Fraction(eps)
        r = 1 / math.sqrt(float(ms))
        x = [Fraction(row[i]) * Fraction(g[i]) for i in range(n)]   # r applied in float at the end
        G = [sum(x[i] * Fraction(Wg[i][j]) for i in range(n)) for j in range(len(Wg[0]))]
        U = [sum(x[i] * Fraction(Wu[i][j]) for i in range(n)) for j in range(len(Wu[0]))]
        if act == "relu":
            h = [max(G[j], 0) * U[j] for j in range(len(G))]      # relu(G r) U r = relu(G) U r^2
        else:
            h = [G[j] * U[j] for j in range(len(G))]
        y = [float(sum(h[j] * Fraction(Wd[j][k]) for j in range(len(h)))) * r * r for k in range(len(Wd[0]))]
        out.append(y)
    return np.array(out)


@pytest.mark.parametrize("act", ["relu", "bilinear"])
def test_glu_brute_force_tiny(act):
    rng = np.random.default_rng(11)
    M, n, f = 3, 5, 6
    a = rng.integers(-9, 10, (M, n)) / 4.0
    Wg = rng.integers(-9, 10, (n, f)) / 8.0
    Wu = rng.integers(-9, 10, (n, f)) / 8.0
    Wd = rng.integers(-9, 10, (f, n)) / 8.0
    g = rng.integers(1, 9, n) / 4.0
    ref = _brute_glu_exact(a.tolist(), Wg.tolist(), Wu.tolist(), Wd.tolist(), g, 0.0625, act)
    np.testing.assert_allclose(O.glu_ffn(a, Wg, Wu, Wd, g, 0.0625, act), ref, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("act", ["silu", "relu", "bilinear"])
@pytest.mark.parametrize("eps", [0.0, 1e-5])
def test_glu_deferred_equals_unoptimized(act, eps):
    """The paper's claim: Fig 3(b)/4(b) compute the same FFN output as Fig 3(a)/4(a)."""
    rng = np.random.default_rng(3)
    M, n, f = 6, 32, 40
    a = rng.standard_normal((M, n)) * rng.uniform(0.1, 10, (M, 1))
    Wg, Wu = rng.standard_normal((n, f)) / np.sqrt(n), rng.standard_normal((n, f)) / np.sqrt(n)
    Wd = rng.standard_normal((f, n)) / np.sqrt(f)
    g = rng.uniform(0.5, 1.5, n)
    y = O.glu_ffn(a, Wg, Wu, Wd, g, eps, act)
    y2 = O.glu_ffn_deferred(a, O.merge_norm_weights(Wg, g), O.merge_norm_weights(Wu, g), Wd, eps, act)
    np.testing.assert_allclose(y2, y, rtol=1e-12, atol=1e-12)


def test_glu_faults_detected():
    """silu applied AFTER the deferred scale (wrong for a non-scale-invariant act) must fail"""
    rng = np.random.default_rng(4)
    a = rng.standard_normal((4, 16)) * 3
    Wg, Wu = rng.standard_normal((16, 8)), rng.standard_normal((16, 8))
    h = O.glu_hidden(a, Wg, Wu, None, 0.0, "silu")
    r = 1.0 / O.rmse(a, 0.0)
    wrong = O.glu_act(a @ Wg, "silu") * (a @ Wu) * (r * r)[:, None]   # Fig 4(b) form used for silu
    assert not np.allclose(wrong, h, rtol=1e-3)


# ---------------------------------------------------------------- RoPE / QKV (NEXT-2)

def _tables(max_pos, h, base=10000.0):
    i = np.arange(h // 2)
    theta = base ** (-2.0 * i / h)
    ang = np.arange(max_pos)[:, None] * theta[None, :]
    return np.cos(ang), np.sin(ang)


def test_rope_worked_quarter_turn():
    """m*theta = pi/2: cos = 0, sin = 1 -> (x1, x2) -> (-x2, x1), the paper's permute"""
    cos_tab = np.array([[1.0], [0.0]])
    sin_tab = np.array([[0.0], [1.0]])
    y = O.rope(np.array([[3.0, 4.0], [3.0, 4.0]]), [0, 1], cos_tab, sin_tab)
    np.testing.assert_array_equal(y, [[3.0, 4.0], [-4.0, 3.0]])
    np.testing.assert_array_equal(O.rope_permute(np.array([1.0, 2.0, 3.0, 4.0])), [-2.0, 1.0, -4.0, 3.0])


def test_rope_is_a_rotation_and_relative():
    """Each pair is rotated by m*theta_i: norms are preserved and q.k after RoPE depends only on
    the relative position (RoPE's defining property) — checked with math.cos/sin per pair."""
    rng = np.random.default_rng(6)
    h, max_pos = 16, 64
    cos_tab, sin_tab = _tables(max_pos, h)
    q, k = rng.standard_normal((1, h)), rng.standard_normal((1, h))
    for m, n in ((5, 3), (40, 1), (7, 7)):
        qm = O.rope(q, [m], cos_tab, sin_tab)
        kn = O.rope(k, [n], cos_tab, sin_tab)
        np.testing.assert_allclose(np.linalg.norm(qm), np.linalg.norm(q), rtol=1e-14)
        rel = O.rope(q, [m - n], cos_tab, sin_tab)
        assert float((qm @ kn.T)[0, 0]) == pytest.approx(float((rel @ k.T)[0, 0]), rel=1e-12, abs=1e-12)
        # explicit 2x2 rotation per pair with math
        for i in range(h // 2):
            ang = m * 10000.0 ** (-2.0 * i / h)
            x1, x2 = q[0, 2 * i], q[0, 2 * i + 1]
            assert qm[0, 2 * i] == pytest.approx(x1 * math.cos(ang) - x2 * math.sin(ang), abs=1e-13)
            assert qm[0, 2 * i + 1] == pytest.approx(x2 * math.cos(ang) + x1 * math.sin(ang), abs=1e-13)


@pytest.mark.parametrize("eps", [0.0, 1e-5])
@pytest.mark.parametrize("qk_scale", [1.0, 1.0 / math.sqrt(math.sqrt(128.0))])
def test_qkv_rope_deferred_equals_unfused(eps, qk_scale):
    """The paper's claim: Fig 5(b) (cos/sin scaled by 1/RMS once per token) == Fig 5(a)"""
    rng = np.random.default_rng(7)
    M, n, h = 5, 48, 8
    n_q, n_k, n_v = 4 * h, 2 * h, 2 * h
    N = n_q + n_k + n_v
    a = rng.standard_normal((M, n)) * rng.uniform(0.1, 5, (M, 1))
    W = rng.standard_normal((n, N)) / np.sqrt(n)
    g = rng.uniform(0.5, 1.5, n)
    cos_tab, sin_tab = _tables(32, h)
    pos = rng.integers(0, 32, M)
    ref = O.qkv_rope_unfused(a, W, g, eps, n_q + n_k, h, pos, cos_tab, sin_tab, qk_scale)
    got = O.qkv_rope_deferred(a, O.merge_norm_weights(W, g), eps, n_q + n_k, h, pos, cos_tab, sin_tab, qk_scale)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    # the scaled dot product: (q' . k') == (rope(q) . rope(k)) / sqrt(h) when qk_scale = h^-1/4
    if qk_scale != 1.0:
        plain = O.qkv_rope_unfused(a, W, g, eps, n_q + n_k, h, pos, cos_tab, sin_tab, 1.0)
        qd = ref[:, :h] @ ref[:, n_q:n_q + h].T
        np.testing.assert_allclose(qd, plain[:, :h] @ plain[:, n_q:n_q + h].T / math.sqrt(128.0), rtol=1e-12)


def test_rope_fault_detected():
    """rotate-half pairing (i, i+h/2) instead of the paper's adjacent pairs must differ"""
    rng = np.random.default_rng(8)
    x = rng.standard_normal((1, 8))
    cos_tab, sin_tab = _tables(4, 8)
    y = O.rope(x, [3], cos_tab, sin_tab)
    c, s = O.rope_cos_sin([3], cos_tab, sin_tab)
    half = np.concatenate([-x[:, 4:], x[:, :4]], axis=1)
    assert not np.allclose(x * c + half * s, y)


# ---------------------------------------------------------------- ReLU FFN (Fig 2)

def test_relu_ffn_worked():
    """a = [3, -4], g = 1, eps = 0: x = a/sqrt(12.5); Wu = I; relu keeps x1; Wd = [[1],[1]]:
    y = 3/sqrt(12.5) (hand-worked, Fig 2(a))"""
    a = np.array([[3.0, -4.0]])
    y = O.relu_ffn(a, np.eye(2), np.array([[1.0], [1.0]]))
    assert y[0, 0] == pytest.approx(3 / math.sqrt(12.5), rel=1e-15)
    h, s = O.relu_ffn_deferred(a, np.eye(2), np.array([[1.0], [1.0]]))
    np.testing.assert_array_equal(h, [[3.0, 0.0]])
    assert s[0] == pytest.approx(1 / math.sqrt(12.5), rel=1e-15)


@pytest.mark.parametrize("eps", [0.0, 1e-5])
def test_relu_ffn_deferred_equals_unoptimized(eps):
    rng = np.random.default_rng(12)
    a = rng.standard_normal((6, 24)) * rng.uniform(0.1, 10, (6, 1))
    Wu, Wd = rng.standard_normal((24, 40)), rng.standard_normal((40, 24))
    g = rng.uniform(0.5, 1.5, 24)
    h, s = O.relu_ffn_deferred(a, O.merge_norm_weights(Wu, g), Wd, eps)
    np.testing.assert_allclose((h @ Wd) * s[:, None], O.relu_ffn(a, Wu, Wd, g, eps), rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- QK-norm + RoPE (NEXT-4 part)

def test_permute_g_definition():
    np.testing.assert_array_equal(O.permute_g(np.array([1.0, 2.0, 3.0, 4.0])), [2.0, 1.0, 4.0, 3.0])


def test_qk_norm_scale_invariance_worked():
    """Fig 6: y = a W* s_a s_c g = a W* s_b g. Worked: head b = [3, 4] (RMS^2 = 12.5); any s_a
    cancels; with g = [2, 1], position 0 (cos 1, sin 0): y = [6, 4] / sqrt(12.5)."""
    a = np.array([[3.0, 4.0]])
    cos_tab, sin_tab = np.array([[1.0]]), np.array([[0.0]])
    for scale in (1.0, 1e-3, 7.0):   # scaling a scales acc; the QK-norm output must not change
        y = O.qk_norm_rope_deferred(a * scale, np.eye(2), 0.0, 2, 0, 2, np.array([2.0, 1.0]), None, 0.0, [0],
                                    cos_tab, sin_tab)
        np.testing.assert_allclose(y[0], np.array([6.0, 4.0]) / math.sqrt(12.5), rtol=1e-14)


@pytest.mark.parametrize("eps_qk", [0.0, 1e-6])
@pytest.mark.parametrize("eps", [0.0, 1e-5])
def test_qk_norm_rope_deferred_equals_unfused(eps, eps_qk):
    """The paper's claim (exact with the eps reading c28): Figs 6(b)+7(b) == Figs 6(a)+7(a)"""
    rng = np.random.default_rng(13)
    M, n, h = 5, 40, 8
    n_q, n_k, n_v = 3 * h, 2 * h, 2 * h
    N = n_q + n_k + n_v
    a = rng.standard_normal((M, n)) * rng.uniform(0.01, 10, (M, 1))
    W = rng.standard_normal((n, N)) / np.sqrt(n)
    g = rng.uniform(0.5, 1.5, n)
    g_q, g_k = rng.uniform(0.5, 1.5, h), rng.uniform(0.5, 1.5, h)
    cos_tab, sin_tab = _tables(16, h)
    pos = rng.integers(0, 16, M)
    ref = O.qk_norm_rope_unfused(a, W, g, eps, n_q, n_k, h, g_q, g_k, eps_qk, pos, cos_tab, sin_tab, 0.7)
    got = O.qk_norm_rope_deferred(a, O.merge_norm_weights(W, g), eps, n_q, n_k, h, g_q, g_k, eps_qk, pos,
                                  cos_tab, sin_tab, 0.7)
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-12)


def test_qk_norm_head_rms_is_one():
    """after the per-head RMSNorm with g = 1 and RoPE (a rotation), each head has RMS 1"""
    rng = np.random.default_rng(14)
    a = rng.standard_normal((3, 16))
    W = rng.standard_normal((16, 32))
    cos_tab, sin_tab = _tables(8, 8)
    y = O.qk_norm_rope_unfused(a, W, None, 0.0, 16, 8, 8, np.ones(8), np.ones(8), 0.0, [1, 2, 3], cos_tab, sin_tab)
    for h0 in range(0, 24, 8):
        np.testing.assert_allclose(np.sqrt(np.mean(y[:, h0:h0 + 8] ** 2, axis=1)), 1.0, rtol=1e-13)


# ---------------------------------------------------------------- NEXT-4: LayerNorm deferred without a foldable V

def _ln_case(seed, M=6, n=64, k=40, mean_scale=3.0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((M, n)) + rng.uniform(-mean_scale, mean_scale, (M, 1))
    W = rng.standard_normal((n, k)) / np.sqrt(n)
    g = rng.uniform(0.5, 1.5, n)
    b = rng.uniform(-0.1, 0.1, n)
    c = rng.uniform(-0.1, 0.1, k)
    return a, W, g, b, c


def test_layernorm_deferred_worked():
    """LayerNorm([1, 3]) = [-1, 1]: with W* = I, u = [1, 1], eps = 0 the deferred
    form gives ([1,3] - 2 [1,1]) / sqrt((1+9)/2 - 2^2) = [-1, 1]."""
    z = O.layernorm_deferred(np.array([[1.0, 3.0]]), np.eye(2), O.column_sums(np.eye(2)), None, 0.0)
    np.testing.assert_array_equal(z, [[-1.0, 1.0]])
    np.testing.assert_array_equal(O.column_sums(np.array([[1.0, 2.0], [3.0, 5.0]])), [4.0, 7.0])


@pytest.mark.parametrize("eps", [0.0, 1e-5])
def test_layernorm_deferred_equals_unfused(eps):
    """(a - mu 1) W* = a W* - mu u: the deferred LayerNorm equals the unfused LayerNorm -> linear
    (PAPER.md:33), which test_layernorm_matches_torch_f64 pins to torch.layer_norm."""
    a, W, g, b, c = _ln_case(21)
    ref = O.norm_linear(a, W, g, b, c, eps, "layernorm")
    Ws, cs = O.fold_weights(W, g, b, c)
    assert O.rowwise_rel_err(O.layernorm_deferred(a, Ws, O.column_sums(Ws), cs, eps), ref) < 1e-11


def test_layernorm_deferred_shift_invariant_and_constant_rows():
    """LayerNorm is invariant to adding a constant to every input (the -mu u term removes it),
    and a constant row (zero variance) with eps > 0 maps to c* exactly."""
    a, W, g, b, c = _ln_case(22)
    Ws, cs = O.fold_weights(W, g, b, c)
    u = O.column_sums(Ws)
    z0 = O.layernorm_deferred(a, Ws, u, cs, 1e-5)
    z1 = O.layernorm_deferred(a + 2.5, Ws, u, cs, 1e-5)
    assert O.rowwise_rel_err(z1, z0) < 1e-10
    zc = O.layernorm_deferred(np.full((2, a.shape[1]), 0.75), Ws, u, cs, 1e-5)
    np.testing.assert_allclose(zc, np.broadcast_to(cs, zc.shape), rtol=0, atol=1e-12)


def test_layernorm_deferred_faults_detected():
    """Plausible mistakes fail the pins above: u from the original W (not W*), mu^2 dropped from
    the variance, the correction sign flipped."""
    a, W, g, b, c = _ln_case(23)
    ref = O.norm_linear(a, W, g, b, c, 1e-5, "layernorm")
    Ws, cs = O.fold_weights(W, g, b, c)
    u = O.column_sums(Ws)
    assert O.rowwise_rel_err(O.layernorm_deferred(a, Ws, O.column_sums(W), cs, 1e-5), ref) > 1e-2
    n = a.shape[1]
    mu = a.mean(axis=1)
    no_mu2 = (a @ Ws - mu[:, None] * u) / np.sqrt((a * a).sum(axis=1) / n + 1e-5)[:, None] + cs
    assert O.rowwise_rel_err(no_mu2, ref) > 1e-2
    flipped = (a @ Ws + mu[:, None] * u) / np.sqrt((a * a).sum(axis=1) / n - mu * mu + 1e-5)[:, None] + cs
    assert O.rowwise_rel_err(flipped, ref) > 1e-2


# ---------------------------------------------------------------- App. B: eliminating 1/n

def test_rss_worked():
    """n = 4, a = [1,1,1,1], W = I, g = 1, eps = 0: RSS = 2, g* = sqrt(4) = 2, z = 2a/2 = a,
    which is RMSNorm(a) = a / RMS(a) = a / 1."""
    Ws, cs = O.fold_weights_rss(np.eye(4))
    np.testing.assert_array_equal(Ws, 2.0 * np.eye(4))
    np.testing.assert_array_equal(O.deferred_linear_rss(np.ones((1, 4)), Ws, cs, 0.0), np.ones((1, 4)))


@pytest.mark.parametrize("eps", [0.0, 1e-5, 1e-2])
def test_rss_equals_rms_path(eps):
    """(a W*_rss)/RSSe(a) = (a W*)/RMSe(a) with g* = sqrt(n) g and RSSe = sqrt(n eps + sum a^2)
    (PAPER.md:196-200), including low-energy rows where eps matters; a fault (eps instead of
    n eps under the root) fails."""
    a, W, g, b, c = _ln_case(24, mean_scale=0.0)
    a[1] *= 1e-3
    ref = O.deferred_linear(a, *O.fold_weights(W, g, b, c)[:1], O.fold_weights(W, g, b, c)[1], eps)
    Wr, cr = O.fold_weights_rss(W, g, b, c)
    assert O.rowwise_rel_err(O.deferred_linear_rss(a, Wr, cr, eps), ref) < 1e-12
    if eps >= 1e-5:
        wrong = (a @ Wr) / np.sqrt(eps + (a * a).sum(axis=1))[:, None] + cr
        assert O.rowwise_rel_err(wrong, ref) > 1e-3
