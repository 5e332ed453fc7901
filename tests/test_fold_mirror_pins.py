"""Pins for oracle/fold_mirror.py (the bit-exact target of the CUDA folds) — CPU only.

The mirror is pinned (a) bit-exactly to the hand-derived worked examples, whose
values are exact in bf16/fp32, and (b) to the plain fp64 folds of the oracle
within the rounding the fold contract states (one fp32 rounding then one bf16
rounding for W*, V*; one fp32 rounding of an fp64 sum for c*, b_prev*).
"""
import numpy as np
import pytest

from oracle import flashnorm_oracle as O
from oracle import fold_mirror as FM
from synth import bf16_bits, bits_to_f32, gen_layer, gen_upstream


def _bits(x):
    return bf16_bits(np.asarray(x, np.float32))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_mirror_worked_examples(golden, dtype):
    for ex in golden["fold_weights"]:
        Wt = np.array(ex["W"], np.float32).T.copy()          # storage is Wt = W^T
        store = _bits(Wt) if dtype == "bf16" else Wt
        g = None if ex["g"] is None else np.array(ex["g"], np.float32)
        b = None if ex["b"] is None else np.array(ex["b"], np.float32)
        c = None if ex["c"] is None else np.array(ex["c"], np.float32)
        Ws, cs = FM.fold_weights(store, g, b, c, dtype)
        Ws_f = bits_to_f32(Ws) if dtype == "bf16" else Ws
        np.testing.assert_array_equal(Ws_f.T, np.array(ex["W_star"], np.float32), err_msg=ex["cite"])
        if ex["c_star"] is not None:
            np.testing.assert_array_equal(cs, np.array(ex["c_star"], np.float32))
    for ex in golden["fold_mean_center"]:
        Vt = np.array(ex["V"], np.float32).T.copy()
        store = _bits(Vt) if dtype == "bf16" else Vt
        bp = None if ex["b_prev"] is None else np.array(ex["b_prev"], np.float32)
        Vs, bs, s = FM.fold_mean_center(store, bp, dtype)
        Vs_f = bits_to_f32(Vs) if dtype == "bf16" else Vs
        np.testing.assert_array_equal(s, np.array(ex["s"], float))
        np.testing.assert_array_equal(Vs_f.T, np.array(ex["V_star"], np.float32), err_msg=ex["cite"])
        if bp is not None:
            np.testing.assert_array_equal(bs, np.array(ex["b_prev_star"], np.float32))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("N,K", [(48, 64), (37, 1000), (130, 4096)])
def test_mirror_fold_weights_vs_fp64(dtype, N, K):
    Wt, g, b, c = gen_layer(3, N, K, dtype, with_b=True, with_c=True)
    store = bf16_bits(Wt) if dtype == "bf16" else Wt
    Ws, cs = FM.fold_weights(store, g, b, c, dtype)
    Ws_f = (bits_to_f32(Ws) if dtype == "bf16" else Ws).astype(np.float64)
    W_exact, c_exact = O.fold_weights(Wt.T.astype(np.float64), g, b, c)
    u = 2.0 ** -8 if dtype == "bf16" else 2.0 ** -24       # unit roundoff of the storage dtype
    rel = np.abs(Ws_f.T - W_exact) / np.maximum(np.abs(W_exact), 1e-30)
    assert rel.max() <= u * (1 + 2.0 ** -15)              # + the fp32 pre-rounding (double rounding)
    np.testing.assert_allclose(cs.astype(np.float64), c_exact, rtol=2.0 ** -24, atol=1e-12)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("n_out,d_in", [(40, 24), (100, 72), (512, 256)])
def test_mirror_fold_mean_center_vs_fp64(dtype, n_out, d_in):
    _, Vt, bp = gen_upstream(4, 2, d_in, n_out, dtype)
    store = bf16_bits(Vt) if dtype == "bf16" else Vt
    Vs, bs, s = FM.fold_mean_center(store, bp, dtype)
    V = Vt.T.astype(np.float64)                                  # paper V: d_in x n_out
    np.testing.assert_allclose(s, O.row_sums(V), rtol=1e-13, atol=1e-12)
    V_exact, b_exact = O.fold_mean_center(V, bp)
    Vs_f = (bits_to_f32(Vs) if dtype == "bf16" else Vs).astype(np.float64).T
    u = 2.0 ** -8 if dtype == "bf16" else 2.0 ** -24
    # contract (reading c21): mu_i = RN_f32(s_i / n), V* = RN_dtype(v - mu_i) in f32.  Error bound of
    # that evaluation against the exact fp64 fold: the mu rounding (<= 2^-24 |mu_i|, carried through
    # the subtraction and the final rounding) plus one rounding of the result (<= u |V*|; for bf16
    # the f32 subtraction's 2^-24 is inside the double-rounding slack)
    mu = np.abs(s / n_out)[:, None]
    bound = u * (1 + 2.0 ** -15) * np.abs(V_exact) + 2.0 ** -24 * mu * (1 + u) * (1 + 2.0 ** -15)
    assert np.all(np.abs(Vs_f - V_exact) <= bound)
    np.testing.assert_allclose(bs.astype(np.float64), b_exact, rtol=2.0 ** -23, atol=1e-7)


def test_mirror_mean_center_identity_holds_after_rounding():
    """x V* + b* ~= mean_center(x V + b_prev) with the mirror's rounded V* (PAPER.md:46-49)."""
    x, Vt, bp = gen_upstream(5, 6, 64, 96, "f32")
    Vs, bs, _ = FM.fold_mean_center(Vt, bp, "f32")
    lhs = x.astype(np.float64) @ Vs.T.astype(np.float64) + bs
    rhs = O.mean_center(O.linear(x, Vt.T, bp))
    np.testing.assert_allclose(lhs, rhs, atol=1e-5)
