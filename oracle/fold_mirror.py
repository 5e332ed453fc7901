"""CPU mirror of the weight folds, in the SAME precision and summation order as
the CUDA fold kernels, so that the GPU folds can be checked BIT-EXACT.

TEST INFRASTRUCTURE ONLY (same import rule as flashnorm_oracle.py).  Written
independently from the CUDA sources: it implements the *contract* stated in
include/flashnorm.h (sections "fold_weights numerics" and "fold_mean_center
numerics"), not the kernels.  It is itself pinned (tests/test_oracle_pins.py)
against the plain fp64 folds of flashnorm_oracle.py (to within the documented
rounding) and against the worked examples in tests/golden/.

North star: "folding is checked bit-exact against a CPU fold done in the same
precision and order" (BASELINE.json:5).  Math: PAPER.md:16 (W* = g_i W_ij),
PAPER.md:25 (c* = c + b W), PAPER.md:44-49 (s_i, V*), reading c7 (b_prev*).
"""
from __future__ import annotations

import numpy as np

LANES = 32            # lanes per row-warp in the c* reduction
CHUNK_BYTES = 16      # one 128-bit access
COLSUM_ROWS = 32      # rows per fp64 partial column sum in fold_mean_center
BPREV_THREADS = 256   # threads in the b_prev mean reduction


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bits (finite values)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _as_f32_values(Wt, dtype):
    """Storage tensor (bf16 bits as uint16, or float32) -> float32 values."""
    if dtype == "bf16":
        return bf16_bits_to_f32(Wt)
    return np.ascontiguousarray(Wt, dtype=np.float32)


def _store(x32: np.ndarray, dtype):
    return f32_to_bf16_bits(x32) if dtype == "bf16" else x32.astype(np.float32)


def fold_weights(Wt, g, b, c, dtype="bf16"):
    """Mirror of flashnorm_fold_weights.

    Wt: [N, K] storage (uint16 bf16 bits, or float32).  g, b: [K] float32 or None;
    c: [N] float32 or None.  Returns (Wt_star in storage dtype, c_star float32 or None).

    W*t[j, i] = RN_dtype( RN_f32(g_i * W_ij) )
    c*_j      = RN_f32( c_j + S_j ),  S_j = fp64 sum of b_i * W_ij (exact fp64
                products) in the lane order: lane l owns 16-byte chunks
                q = l, l+32, ... (ascending), elements ascending inside a chunk;
                the 32 lane sums are combined by the xor butterfly 16,8,4,2,1.
                                                               
    """
    w = _as_f32_values(Wt, dtype)
    N, K = w.shape
    if g is None:
        wstar = w.copy()
    else:
        wstar = (np.asarray(g, np.float32)[None, :] * w).astype(np.float32)  # IEEE RN product
    Wt_star = _store(wstar, dtype)

    if b is None and c is None:
        return Wt_star, None
    if b is None:
        return Wt_star, np.asarray(c, np.float32).copy()

    E = CHUNK_BYTES // (2 if dtype == "bf16" else 4)
    nchunks = -(-K // E)
    rounds = -(-nchunks // LANES)
    p = np.asarray(b, np.float64)[None, :] * w.astype(np.float64)          # exact in fp64
    pad = np.zeros((N, rounds * LANES * E), np.float64)
    pad[:, :K] = p
    p = pad.reshape(N, rounds, LANES, E)
    acc = np.zeros((N, LANES), np.float64)
    for r in range(rounds):
        for e in range(E):
            acc = acc + p[:, r, :, e]
    idx = np.arange(LANES)
    for off in (16, 8, 4, 2, 1):
        acc = acc + acc[:, idx ^ off]
    S = acc[:, 0]
    c64 = np.zeros(N) if c is None else np.asarray(c, np.float32).astype(np.float64)
    c_star = (c64 + S).astype(np.float32)
    return Wt_star, c_star


def fold_mean_center(Vt, b_prev, dtype="bf16"):
    """Mirror of flashnorm_fold_mean_center.

    Vt: [n_out, d_in] storage (paper V = Vt.T, d_in x n_out).  Returns
    (Vt_star storage, b_prev_star float32 or None, s float64[d_in]).

    partial[c, i] = fp64 sum over rows j in [32c, 32c+32) ascending of Vt[j, i]
    s_i           = lane l sums partial[c, i], c = l, l+32, ... ascending; the 32 lane
                    sums are combined by the xor butterfly 16,8,4,2,1
    mu_i          = RN_f32( s_i / n_out )   (fp64 quotient, rounded once)
    V*t[j, i]     = RN_dtype( Vt[j, i] -_f32 mu_i )  (one float32 subtraction, reading c21)
    b_prev*_j     = RN_f32( b_prev_j - mean ), mean = T / n_out where thread t of
                    256 sums j = t, t+256, ... ascending, each warp of 32 threads
                    xor-butterflies (16,8,4,2,1) and T = sum of the 8 warp totals
                    in ascending warp order.                          (reading c7)
    """
    v = _as_f32_values(Vt, dtype).astype(np.float64)
    n_out, d_in = v.shape
    nchunk = -(-n_out // COLSUM_ROWS)
    partial = np.zeros((nchunk, d_in))
    for ci in range(nchunk):
        acc = np.zeros(d_in)
        for j in range(ci * COLSUM_ROWS, min((ci + 1) * COLSUM_ROWS, n_out)):
            acc = acc + v[j]
        partial[ci] = acc
    rounds = -(-nchunk // LANES)
    padp = np.zeros((rounds * LANES, d_in))
    padp[:nchunk] = partial
    lane_acc = np.zeros((LANES, d_in))
    for r in range(rounds):
        lane_acc = lane_acc + padp[r * LANES:(r + 1) * LANES]
    idx = np.arange(LANES)
    for off in (16, 8, 4, 2, 1):
        lane_acc = lane_acc + lane_acc[idx ^ off]
    s = lane_acc[0]
    mu = (s / float(n_out)).astype(np.float32)                 # RN_f32 of the fp64 quotient
    vstar = _as_f32_values(Vt, dtype) - mu[None, :]             # one IEEE float32 subtraction
    Vt_star = _store(vstar, dtype)

    bstar = None
    if b_prev is not None:
        bp = np.asarray(b_prev, np.float32).astype(np.float64)
        T = BPREV_THREADS
        rounds = -(-n_out // T)
        pad = np.zeros(rounds * T)
        pad[:n_out] = bp
        acc = np.zeros(T)
        for r in range(rounds):
            acc = acc + pad[r * T:(r + 1) * T]
        acc = acc.reshape(T // LANES, LANES)
        idx = np.arange(LANES)
        for off in (16, 8, 4, 2, 1):
            acc = acc + acc[:, idx ^ off]
        total = 0.0
        for w in range(T // LANES):
            total = total + acc[w, 0]
        mean = total / float(n_out)
        bstar = (bp - mean).astype(np.float32)
    return Vt_star, bstar, s
