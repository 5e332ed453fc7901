"""FlashNorm oracle: plain, slow, obviously-correct fp64 CPU definitions.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2407_09577_b200``) never imports it and
shares no code with it.

Every function follows a passage of /root/reference/PAPER.md (arXiv 2407.09577,
"FlashNorm: fast normalization for LLMs"), cited as PAPER.md:<line> (section).
Where the paper is silent the reading taken is the one listed in DESIGN.md
("Readings of the paper"), cited here as [reading cN].

Conventions
-----------
* fp64 throughout (numpy float64); the only library primitive used as a step
  is the matrix product ``@`` ("vector-matrix multiplication").
* Paper convention for weights: ``W`` is n x k with ``y = x W``,
  i.e. rows index the *input* features.  The CUDA boundary stores the
  transpose ``Wt`` (N x K); callers pass ``Wt.T``.
* Activations are a batch of row vectors ``a[M, n]``; RMS is per row
  (PAPER.md:14 defines it per vector).

Pins: tests/test_oracle_pins.py pins every function here to values/identities
fixed by the paper and by mathematics (tests/golden/*.json).  DyT's elementwise
formula is not stated by the paper: ``dyt`` is pinned only to reading c10
("parity pinned to the stated reading").
"""
from __future__ import annotations

import numpy as np

MODES = ("rmsnorm", "layernorm", "dyt")


def _f64(x):
    return None if x is None else np.asarray(x, dtype=np.float64)


# ---------------------------------------------------------------------------
# RMS and its variants
# ---------------------------------------------------------------------------

def rms(a):
    """RMS(a) = sqrt((1/n) sum_i a_i^2) per row.  PAPER.md:14 (§1)."""
    a = _f64(a)
    n = a.shape[-1]
    return np.sqrt(np.sum(a * a, axis=-1) / n)


def rmse(a, eps):
    """RMSe(a) = sqrt(eps + (1/n) sum_i a_i^2).  PAPER.md:177 (App. A) [reading c1]."""
    a = _f64(a)
    n = a.shape[-1]
    return np.sqrt(eps + np.sum(a * a, axis=-1) / n)


def rss(a):
    """RSS(a) = sqrt(sum_i a_i^2).  PAPER.md:185-187 (App. B)."""
    a = _f64(a)
    return np.sqrt(np.sum(a * a, axis=-1))


def rsse(a, eps):
    """RSSe(a) = sqrt(n eps + sum_i a_i^2).  PAPER.md:196-200 (App. B)."""
    a = _f64(a)
    n = a.shape[-1]
    return np.sqrt(n * eps + np.sum(a * a, axis=-1))


def mean_square(a):
    """MS(a) = (1/n) sum a_i^2 = RMS(a)^2.  PAPER.md:70-73 (§2.2)."""
    a = _f64(a)
    return np.sum(a * a, axis=-1) / a.shape[-1]


# ---------------------------------------------------------------------------
# Normalizations (unfused, Fig 1(a))
# ---------------------------------------------------------------------------

def rmsnorm(a, g=None, b=None, eps=0.0):
    """y_i = a_i / RMSe(a) * g_i (+ b_i).

    PAPER.md:14 (§1) for y_i = a_i/RMS * g_i; PAPER.md:177 (App. A) for eps;
    the optional bias b "right after scaling by weights g_i" PAPER.md:25 (§1.1).
    """
    a = _f64(a)
    y = a / rmse(a, eps)[..., None]
    if g is not None:
        y = y * _f64(g)
    if b is not None:
        y = y + _f64(b)
    return y


def mean_center(y):
    """a_j = y_j - mu, mu = (1/n) sum_j y_j.  PAPER.md:40, 45 (§1.2)."""
    y = _f64(y)
    return y - np.mean(y, axis=-1, keepdims=True)


def layernorm(a, g=None, b=None, eps=0.0):
    """LayerNorm = mean centering followed by RMSNorm.  PAPER.md:33 (§1.2) [reading c8]."""
    return rmsnorm(mean_center(a), g, b, eps)


def dyt(a, g=None, b=None, alpha=0.5):
    """DyT: y = g * tanh(alpha * a) + b.

    The paper names DyT and its bias b after g but
    never states the elementwise formula: [reading c10].
    """
    a = _f64(a)
    y = np.tanh(alpha * a)
    if g is not None:
        y = y * _f64(g)
    if b is not None:
        y = y + _f64(b)
    return y


def normalize(a, mode, g=None, b=None, eps=0.0, alpha=0.5):
    if mode == "rmsnorm":
        return rmsnorm(a, g, b, eps)
    if mode == "layernorm":
        return layernorm(a, g, b, eps)
    if mode == "dyt":
        return dyt(a, g, b, alpha)
    raise ValueError(f"mode must be one of {MODES}, got {mode!r}")


# ---------------------------------------------------------------------------
# Linear layer and the unfused norm -> linear path (Fig 1(a))
# ---------------------------------------------------------------------------

def linear(y, W, c=None):
    """z = y W (+ c).  W is n x k (paper convention)."""
    z = _f64(y) @ _f64(W)
    if c is not None:
        z = z + _f64(c)
    return z


def norm_linear(a, W, g=None, b=None, c=None, eps=0.0, mode="rmsnorm", alpha=0.5):
    """Unfused reference: z = Norm(a; g, b) W + c.  Fig 1(a).

    This is what the CUDA path must equal (FlashNorm is "exact");
    it never folds anything.
    """
    return linear(normalize(a, mode, g, b, eps, alpha), W, c)


def upstream_layernorm_linear(x, V, b_prev, W, g=None, b=None, c=None, eps=0.0):
    """Config 4 unfused: a = x V + b_prev, then LayerNorm(a; g, b) W + c.

    PAPER.md:33 (Fig B(a)): linear layer V followed by mean centering and RMSNorm.
    """
    a = linear(x, V, b_prev)
    return norm_linear(a, W, g, b, c, eps, "layernorm")


# ---------------------------------------------------------------------------
# The FlashNorm transforms, written out in fp64 (used to check the paper's
# identities and as the exact target of the folded CUDA tensors)
# ---------------------------------------------------------------------------

def eliminate_norm_bias(W, b=None, c=None):
    """c* = c + b W, with the ORIGINAL W (bias moved before the g merge).

    PAPER.md:25 (§1.1, Fig A(b)) [reading c5].
    """
    W = _f64(W)
    k = W.shape[1]
    cstar = np.zeros(k) if c is None else _f64(c).copy()
    if b is not None:
        cstar = cstar + _f64(b) @ W
    return cstar


def merge_norm_weights(W, g=None):
    """W*_{i,j} = g_i W_{i,j}.  PAPER.md:16 (§1, Fig 1(b))."""
    W = _f64(W)
    if g is None:
        return W.copy()
    return _f64(g)[:, None] * W


def fold_weights(W, g=None, b=None, c=None):
    """(W*, c*) in the paper's order: Fig A first, then Fig 1(b)."""
    return merge_norm_weights(W, g), eliminate_norm_bias(W, b, c)


def deferred_linear(a, Wstar, cstar=None, eps=0.0):
    """Deferred normalization z = (a W*) * 1/RMSe(a) (+ c*, added AFTER scaling).

    PAPER.md:17 (§1, Fig 1(c)): "normalization ... must be done before adding
    the bias" [reading c4]; eps per App. A.
    """
    a = _f64(a)
    z = (a @ _f64(Wstar)) / rmse(a, eps)[..., None]
    if cstar is not None:
        z = z + _f64(cstar)
    return z


def row_sums(V):
    """s_i = sum_j v_{i,j} (sum of row i of V).  PAPER.md:44 (§1.2)."""
    return np.sum(_f64(V), axis=1)


def mean_via_s(x, V):
    """mu = (1/n) sum_i x_i s_i.  PAPER.md:42 (§1.2); n = number of outputs of V [reading c6]."""
    V = _f64(V)
    n = V.shape[1]
    return (_f64(x) @ row_sums(V)) / n


def fold_mean_center(V, b_prev=None):
    """V*_{i,j} = v_{i,j} - s_i / n.  PAPER.md:49 (§1.2, Fig B(b)).

    V's own bias (the paper is silent): b_prev* = b_prev - mean(b_prev) [reading c7].
    """
    V = _f64(V)
    n = V.shape[1]
    Vstar = V - row_sums(V)[:, None] / n
    bstar = None if b_prev is None else _f64(b_prev) - np.mean(_f64(b_prev))
    return Vstar, bstar


# ---------------------------------------------------------------------------
# FFN with a GLU variant (§2.2, Figs 3-4) — NEXT-1
# ---------------------------------------------------------------------------

def relu_ffn(a, Wu, Wd, g=None, eps=0.0):
    """FFN with ReLU, unoptimized Fig 2(a): y = ReLU(RMSNorm(a; g) Wu) Wd (bias-free)."""
    return np.maximum(rmsnorm(a, g, None, eps) @ _f64(Wu), 0.0) @ _f64(Wd)


def relu_ffn_deferred(a, Wu_star, Wd, eps=0.0):
    """Fig 2(b): the normalization deferred to the FFN output, y = (ReLU(a Wu*) Wd) / RMSe(a)
    ("multiplying its argument by a non-negative scaling factor s is the same as scaling its
    output by s").  Returns (h, s) with y = (h Wd) * s."""
    h = np.maximum(_f64(a) @ _f64(Wu_star), 0.0)
    return h, 1.0 / rmse(a, eps)


GLU_ACTS = ("silu", "relu", "bilinear")


def glu_act(x, act):
    """The GLU variant's activation [reading c24]: SwiGLU silu(x) = x / (1 + e^-x),
    ReGLU relu(x) = max(x, 0), bilinear GLU: identity (PAPER.md:70 names ReGLU and
    bilinear GLU; the FFN "with a GLU variant" of Fig 3 is SwiGLU in Llama)."""
    x = _f64(x)
    if act == "silu":
        return x / (1.0 + np.exp(-x))
    if act == "relu":
        return np.maximum(x, 0.0)
    if act == "bilinear":
        return x.copy()
    raise ValueError(act)


def glu_hidden(a, Wg, Wu, g=None, eps=0.0, act="silu"):
    """Unoptimized Fig 3(a) / Fig 4(a): x = RMSNorm(a; g), h = act(x Wg) * (x Wu).

    Bias-free FFN ("bias-free FFNs").  Wg, Wu are n x f (paper convention).
    """
    x = rmsnorm(a, g, None, eps)
    return glu_act(x @ _f64(Wg), act) * (x @ _f64(Wu))


def glu_ffn(a, Wg, Wu, Wd, g=None, eps=0.0, act="silu"):
    """Full FFN output y = h Wd (Fig 3(a)), Wd is f x n."""
    return glu_hidden(a, Wg, Wu, g, eps, act) @ _f64(Wd)


def glu_hidden_deferred(a, Wg_star, Wu_star, eps=0.0, act="silu"):
    """Optimized forms, step by step as the figures draw them [reading c25]:

    Fig 3(b) (silu):  h' = act((a Wg*) / RMSe(a)) * (a Wu*),  output scale s = 1/RMSe(a)
                      ("one set [of f multipliers] can be deferred to the FFN output").
    Fig 4(b) (relu, bilinear): h'' = act(a Wg*) * (a Wu*),   s = 1/MSe(a) = 1/RMSe(a)^2
                      ("eliminate the scaling before the activation function and
                      combine it with the scaling at the output").
    The FFN output is then y = (h Wd) * s.  Returns (h, s[M]).
    """
    a = _f64(a)
    G = a @ _f64(Wg_star)
    U = a @ _f64(Wu_star)
    r = 1.0 / rmse(a, eps)
    if act == "silu":
        return glu_act(G * r[:, None], act) * U, r
    return glu_act(G, act) * U, r * r


def glu_ffn_deferred(a, Wg_star, Wu_star, Wd, eps=0.0, act="silu"):
    """y = (h Wd) * s with (h, s) from glu_hidden_deferred (Fig 3(b) / Fig 4(b) output scaling)."""
    h, s = glu_hidden_deferred(a, Wg_star, Wu_star, eps, act)
    return (h @ _f64(Wd)) * s[:, None]


# ---------------------------------------------------------------------------
# Q/K/V projection with RoPE (§3, Fig 5) — NEXT-2
# ---------------------------------------------------------------------------

def rope_permute(x):
    """permute(x) = (-x2, x1, -x4, x3, ..., -x_h, x_{h-1}) over the last axis."""
    x = _f64(x)
    y = np.empty_like(x)
    y[..., 0::2] = -x[..., 1::2]
    y[..., 1::2] = x[..., 0::2]
    return y


def rope_cos_sin(pos, cos_tab, sin_tab):
    """cos_m = (cos m t1, cos m t1, cos m t2, cos m t2, ...) for each row's position m
    (PAPER.md:87-88); the tables hold cos(m t_i) / sin(m t_i) as [max_pos, h/2] [reading c26]."""
    c = _f64(cos_tab)[np.asarray(pos)]
    s = _f64(sin_tab)[np.asarray(pos)]
    return np.repeat(c, 2, axis=-1), np.repeat(s, 2, axis=-1)


def rope(x, pos, cos_tab, sin_tab):
    """y = x * cos_m + permute(x) * sin_m for one head x[M, h]."""
    c, s = rope_cos_sin(pos, cos_tab, sin_tab)
    return _f64(x) * c + rope_permute(x) * s


def qkv_rope_unfused(a, W, g, eps, n_rope, h, pos, cos_tab, sin_tab, qk_scale=1.0):
    """Fig 5(a): x = RMSNorm(a; g); [Q | K | V] = x W (W is n x N, Q and K in the first n_rope
    columns, h columns per head); RoPE on every Q/K head; Q and K times qk_scale (the paper folds
    sqrt(1/sqrt(h)) of the scaled dot-product into both); V unchanged."""
    y = rmsnorm(a, g, None, eps) @ _f64(W)
    out = y.copy()
    for h0 in range(0, n_rope, h):
        out[:, h0:h0 + h] = rope(y[:, h0:h0 + h], pos, cos_tab, sin_tab) * qk_scale
    return out


def qkv_rope_deferred(a, Wstar, eps, n_rope, h, pos, cos_tab, sin_tab, qk_scale=1.0):
    """Fig 5(b), step by step: acc = a W*; the cos/sin vectors are scaled ONCE per token by
    1/RMSe(a) (and by qk_scale) and shared by all heads; V keeps the explicit 1/RMSe scale
    (PAPER.md:89-93)."""
    acc = _f64(a) @ _f64(Wstar)
    r = 1.0 / rmse(a, eps)
    c, s = rope_cos_sin(pos, cos_tab, sin_tab)
    c = c * (r * qk_scale)[:, None]
    s = s * (r * qk_scale)[:, None]
    out = acc * r[:, None]
    for h0 in range(0, n_rope, h):
        x = acc[:, h0:h0 + h]
        out[:, h0:h0 + h] = x * c + rope_permute(x) * s
    return out


# ---------------------------------------------------------------------------
# QK-normalization with RoPE (§4, Figs 6-7) — NEXT-4 (part)
# ---------------------------------------------------------------------------

def permute_g(g):
    """permuteg(g) = (g2, g1, g4, g3, ..., g_h, g_{h-1})."""
    g = _f64(g)
    y = np.empty_like(g)
    y[0::2] = g[1::2]
    y[1::2] = g[0::2]
    return y


def qk_norm_rope_unfused(a, W, g, eps, n_q, n_k, h, g_q, g_k, eps_qk, pos, cos_tab, sin_tab, qk_scale=1.0):
    """Fig 6(a) + Fig 7(a): x = RMSNorm(a; g, eps); [Q|K|V] = x W; every Q head
    RMSNorm(q; g_q, eps_qk) then RoPE, every K head RMSNorm(k; g_k, eps_qk) then RoPE (OpenELM's
    q_norm_weight / k_norm_weight, the same for all heads of the layer);
    Q, K times qk_scale; V unchanged."""
    y = rmsnorm(a, g, None, eps) @ _f64(W)
    out = y.copy()
    for h0 in range(0, n_q + n_k, h):
        gn = g_q if h0 < n_q else g_k
        qh = rmsnorm(y[:, h0:h0 + h], gn, None, eps_qk)
        out[:, h0:h0 + h] = rope(qh, pos, cos_tab, sin_tab) * qk_scale
    return out


def qk_norm_rope_deferred(a, Wstar, eps, n_q, n_k, h, g_q, g_k, eps_qk, pos, cos_tab, sin_tab, qk_scale=1.0):
    """Fig 6(b) + Fig 7(b), step by step:
    * acc = a W* (no 1/RMS(a) on the Q/K path: s_a cancels, "s_c = s_b / s_a");
    * s_b = 1/RMS of each Q/K head of acc — with eps kept exact as 1/sqrt(MS(acc_head) +
      eps_qk * MSe(a)) [reading c28] (= the paper's 1/RMS(b) when eps_qk = 0);
    * RoPE with the head norm weights fused into cos/sin, shared by all heads:
      y = b s_b * (cos * g) + permute(b) s_b * (sin * permuteg(g));
    * V: acc / RMSe(a)."""
    a = _f64(a)
    acc = a @ _f64(Wstar)
    mse_a = rmse(a, eps) ** 2
    out = acc / np.sqrt(mse_a)[:, None]
    c, s = rope_cos_sin(pos, cos_tab, sin_tab)
    for h0 in range(0, n_q + n_k, h):
        gn = _f64(g_q if h0 < n_q else g_k)
        b = acc[:, h0:h0 + h]
        sb = 1.0 / np.sqrt(np.mean(b * b, axis=1) + eps_qk * mse_a)
        out[:, h0:h0 + h] = (b * (c * gn) + rope_permute(b) * (s * permute_g(gn))) * (sb * qk_scale)[:, None]
    return out


# ---------------------------------------------------------------------------
# LayerNorm deferred past the contraction without a foldable V (NEXT-4) and
# the App. B 1/n elimination
# ---------------------------------------------------------------------------

def column_sums(Wstar):
    """u_j = sum_i W*_{i,j}: the sum of column j of the FOLLOWING layer's weights.

    The §1.2 derivation moves the mean through a linear layer by summing
    weights over the dimension the mean runs over; applied to the layer AFTER the centering,
    (a - mu 1) W* = a W* - mu (1^T W*), the sums run over W*'s input index i [reading c29]."""
    return np.sum(_f64(Wstar), axis=0)


def layernorm_deferred(a, Wstar, u, cstar=None, eps=0.0):
    """LayerNorm -> linear with BOTH the mean centering and the normalization deferred past the
    contraction [reading c29], step by step:
      mu   = (1/n) sum_i a_i                         (the mean)
      acc  = a W*                                    (raw a: nothing before the contraction)
      MS   = (1/n) sum_i (a_i - mu)^2 = (1/n) sum_i a_i^2 - mu^2
                                                     (LayerNorm = mean centering then RMSNorm)
      z    = (acc - mu u) / sqrt(MS + eps) + c*      (u = column_sums(W*); scale before bias)
    """
    a = _f64(a)
    n = a.shape[-1]
    mu = np.sum(a, axis=-1) / n
    acc = a @ _f64(Wstar)
    ms = np.sum(a * a, axis=-1) / n - mu * mu
    z = (acc - mu[:, None] * _f64(u)[None, :]) / np.sqrt(ms + eps)[:, None]
    if cstar is not None:
        z = z + _f64(cstar)
    return z


def fold_weights_rss(W, g=None, b=None, c=None):
    """App. B: g* = sqrt(n) g merged into W: W*_{i,j} = sqrt(n) g_i W_{i,j};
    c* = c + b W as in Fig A (the bias is unaffected by the 1/n elimination)."""
    W = _f64(W)
    n = W.shape[0]
    gs = np.sqrt(n) * (np.ones(n) if g is None else _f64(g))
    return gs[:, None] * W, eliminate_norm_bias(W, b, c)


def deferred_linear_rss(a, Wstar_rss, cstar=None, eps=0.0):
    """z = (a W*_rss) / RSSe(a) + c*, RSSe(a) = sqrt(n eps + sum a_i^2)."""
    a = _f64(a)
    z = (a @ _f64(Wstar_rss)) / rsse(a, eps)[..., None]
    if cstar is not None:
        z = z + _f64(cstar)
    return z


# ---------------------------------------------------------------------------
# Parity metric [reading c12]
# ---------------------------------------------------------------------------

def rowwise_rel_err(z, zref):
    """max_m ||z_m - zref_m||_inf / ||zref_m||_inf  (SPEC.md:432 style, per row)."""
    z = np.asarray(z, dtype=np.float64)
    zref = np.asarray(zref, dtype=np.float64)
    num = np.max(np.abs(z - zref), axis=-1)
    den = np.maximum(np.max(np.abs(zref), axis=-1), 1e-30)
    return float(np.max(num / den)) if num.size else 0.0
