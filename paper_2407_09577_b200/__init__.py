"""paper_2407_09577_b200 — B200-native FlashNorm (arXiv 2407.09577) hot path.

Thin ctypes binding over ``libflashnorm.so`` (the C ABI in include/flashnorm.h).
The names follow the ABI:

* :func:`fold_weights`      — W* = diag(g) W, c* = c + b W
* :func:`fold_mean_center`  — V*_{ij} = V_{ij} - s_i / n
* :func:`linear`            — z = (a W*) / RMSe(a) + c*
* :func:`baseline_norm`     — measurement-only unfused normalization (Fig 1(a))
* :func:`gather_columns`    — column-shard permute after an all-gather

This module only marshals arguments: every step runs in the library's CUDA
kernels.  PyTorch supplies device memory and streams.  There is no CPU
fallback: a missing library or a non-CUDA tensor raises :class:`FlashNormError`.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

__all__ = [
    "FlashNormError", "lib", "lib_path", "fold_weights", "fold_mean_center", "fold_mean_center_workspace_bytes",
    "linear", "linear_from_host", "baseline_norm", "gather_columns", "launch_count", "reset_launch_count",
    "version", "linear_workspace_bytes", "fold_glu_weights", "glu_linear", "linear_scaled", "glu_ffn", "qkv_rope_linear", "relu_ffn_up", "qk_norm_rope_linear",
    "fold_colsum", "layernorm_linear", "linear_gather", "comm_unique_id", "comm_init", "comm_destroy",
    "allgather_columns",
    "MODES", "GLU_ACTS", "PATHS", "EXPORTS",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libflashnorm.so")

MODES = {"rmsnorm": 0, "layernorm": 1, "dyt": 2, "none": 3}
GLU_ACTS = {"silu": 0, "relu": 1, "bilinear": 2}
PATHS = {"auto": 0, "gemm": 1, "gemv": 2, "simt": 3, "gemm1": 4, "gemv_mma": 5}
_DT_BF16, _DT_F32 = 0, 1

# every symbol include/flashnorm.h declares
EXPORTS = [
    "flashnorm_fold_weights", "flashnorm_fold_mean_center_workspace_bytes", "flashnorm_fold_mean_center",
    "flashnorm_linear", "flashnorm_linear_ex", "flashnorm_linear_workspace_bytes", "flashnorm_linear_ws",
    "flashnorm_linear_from_host", "flashnorm_fold_glu_weights", "flashnorm_glu_linear", "flashnorm_linear_scaled",
    "flashnorm_fold_colsum", "flashnorm_layernorm_linear", "flashnorm_linear_gather",
    "flashnorm_comm_unique_id", "flashnorm_comm_init", "flashnorm_comm_destroy",
    "flashnorm_allgather_workspace_bytes", "flashnorm_allgather_columns",
    "flashnorm_qkv_rope_linear", "flashnorm_relu_ffn_up", "flashnorm_qk_norm_rope_linear", "flashnorm_baseline_norm",
    "flashnorm_gather_columns", "flashnorm_status_string", "flashnorm_last_error", "flashnorm_launch_count",
    "flashnorm_reset_launch_count", "flashnorm_version",
]


class FlashNormError(RuntimeError):
    """A libflashnorm call returned a non-OK fn_status (or the library is missing)."""

    def __init__(self, status: int, name: str, msg: str):
        super().__init__(f"{name}: {msg}")
        self.status = status


_LIB = None
_vp, _i64, _f32, _int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_float, ctypes.c_int


def lib() -> ctypes.CDLL:
    """Load libflashnorm.so (built in-tree by paper_2407_09577_b200.build)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(lib_path):
        raise FlashNormError(-1, "load", f"{lib_path} not found: run `python -m paper_2407_09577_b200.build` "
                                         "(there is no CPU fallback)")
    L = ctypes.CDLL(lib_path)
    sig = {
        "flashnorm_fold_weights": [_vp, _i64, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp],
        "flashnorm_fold_mean_center_workspace_bytes": [_i64, _i64],
        "flashnorm_fold_mean_center": [_vp, _i64, _i64, _int, _vp, _vp, _vp, _vp, _vp],
        "flashnorm_linear": [_vp, _vp, _vp, _i64, _i64, _i64, _f32, _f32, _int, _int, _vp, _vp],
        "flashnorm_linear_ex": [_vp, _vp, _vp, _i64, _i64, _i64, _f32, _f32, _int, _int, _vp, _int, _vp],
        "flashnorm_linear_workspace_bytes": [_i64, _i64, _i64, _int, _int, _int],
        "flashnorm_linear_ws": [_vp, _vp, _vp, _i64, _i64, _i64, _f32, _f32, _int, _int, _vp, _int, _vp, _i64, _vp],
        "flashnorm_fold_glu_weights": [_vp, _vp, _i64, _i64, _int, _vp, _vp, _vp],
        "flashnorm_glu_linear": [_vp, _vp, _i64, _i64, _i64, _f32, _int, _int, _vp, _vp, _vp],
        "flashnorm_qkv_rope_linear": [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _f32, _f32, _int, _vp,
                                      _vp],
        "flashnorm_qk_norm_rope_linear": [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _f32, _vp, _vp,
                                          _vp, _f32, _f32, _int, _vp, _vp],
        "flashnorm_relu_ffn_up": [_vp, _vp, _i64, _i64, _i64, _f32, _int, _vp, _vp, _vp],
        "flashnorm_linear_scaled": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _vp, _vp],
        "flashnorm_fold_colsum": [_vp, _i64, _i64, _int, _vp, _vp],
        "flashnorm_comm_unique_id": [_vp],
        "flashnorm_comm_init": [_vp, _int, _int, ctypes.POINTER(ctypes.c_void_p)],
        "flashnorm_comm_destroy": [_vp],
        "flashnorm_allgather_workspace_bytes": [_i64, _i64, _i64, _int],
        "flashnorm_allgather_columns": [_vp, _i64, _i64, _int, _vp, _vp, _vp, _vp],
        "flashnorm_linear_gather": [_vp, _vp, _vp, _i64, _i64, _i64, _f32, _f32, _int, _int, _vp, _int, _i64, _i64,
                                    _vp],
        "flashnorm_layernorm_linear": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _f32, _int, _vp, _vp],
        "flashnorm_linear_from_host": [_vp, _vp, _vp, _i64, _i64, _i64, _f32, _f32, _int, _int, _vp, _vp, _vp,
                                       _vp],
        "flashnorm_baseline_norm": [_vp, _vp, _vp, _i64, _i64, _f32, _int, _f32, _int, _vp, _vp],
        "flashnorm_gather_columns": [_vp, _i64, _i64, _i64, _int, _vp, _vp],
        "flashnorm_status_string": [_int],
        "flashnorm_last_error": [],
        "flashnorm_launch_count": [],
        "flashnorm_reset_launch_count": [],
        "flashnorm_version": [],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = _int
    L.flashnorm_fold_mean_center_workspace_bytes.restype = _i64
    L.flashnorm_linear_workspace_bytes.restype = _i64
    L.flashnorm_allgather_workspace_bytes.restype = _i64
    L.flashnorm_launch_count.restype = _i64
    L.flashnorm_reset_launch_count.restype = None
    for name in ("flashnorm_status_string", "flashnorm_last_error", "flashnorm_version"):
        getattr(L, name).restype = ctypes.c_char_p
    _LIB = L
    return L


def _check(status: int, name: str):
    if status != 0:
        L = lib()
        raise FlashNormError(status, name, f"{L.flashnorm_status_string(status).decode()}: "
                                           f"{L.flashnorm_last_error().decode()}")


# ------------------------------------------------------------------ torch marshalling

def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.bfloat16:
        return _DT_BF16
    if t.dtype == torch.float32:
        return _DT_F32
    raise FlashNormError(3, "dtype", f"unsupported tensor dtype {t.dtype} (bf16 or f32)")


def _dev(t, name: str):
    if t is None:
        return None
    if not t.is_cuda:
        raise FlashNormError(1, name, f"{name} must be a CUDA tensor (no CPU fallback), got device {t.device}")
    if not t.is_contiguous():
        raise FlashNormError(2, name, f"{name} must be contiguous, got strides {tuple(t.stride())}")
    return t


def _vec(t, name: str, n: int):
    torch = _torch()
    if t is None:
        return None
    _dev(t, name)
    if t.dtype != torch.float32 or t.dim() != 1 or t.shape[0] != n:
        raise FlashNormError(2, name, f"{name} must be float32[{n}], got {t.dtype}{list(t.shape)}")
    return t


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(t):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


# ------------------------------------------------------------------ public API

def fold_weights(Wt, g=None, b=None, c=None, out=None, c_out=None):
    """Fold norm weights g and norm bias b into (W*t, c*).  Wt: [N, K] (nn.Linear layout).

    PAPER.md:25 (c* = c + b W, original W) then PAPER.md:16 (W*_ij = g_i W_ij).
    Returns (Wt_star [N, K] same dtype, c_star float32[N] or None).
    """
    torch = _torch()
    _dev(Wt, "Wt")
    if Wt.dim() != 2:
        raise FlashNormError(2, "fold_weights", f"Wt must be 2-D [N, K], got {list(Wt.shape)}")
    N, K = Wt.shape
    g, b, c = _vec(g, "g", K), _vec(b, "b", K), _vec(c, "c", N)
    Ws = out if out is not None else torch.empty_like(Wt)
    cs = c_out
    if cs is None and (b is not None or c is not None):
        cs = torch.empty(N, dtype=torch.float32, device=Wt.device)
    _check(lib().flashnorm_fold_weights(_ptr(Wt), N, K, _dtype_code(Wt), _ptr(g), _ptr(b), _ptr(c), _ptr(Ws),
                                        _ptr(cs), _stream(Wt)), "fold_weights")
    return Ws, cs


def fold_mean_center_workspace_bytes(n_out: int, d_in: int) -> int:
    return int(lib().flashnorm_fold_mean_center_workspace_bytes(n_out, d_in))


def fold_mean_center(Vt, b_prev=None, out=None, workspace=None):
    """Fold LayerNorm's mean centering into the preceding layer.  Vt: [n_out, d_in].

    PAPER.md:42-49: v*_ij = v_ij - s_i/n; b_prev* = b_prev - mean(b_prev) (reading c7).
    Returns (Vt_star, b_prev_star or None).
    """
    torch = _torch()
    _dev(Vt, "Vt")
    n_out, d_in = Vt.shape
    b_prev = _vec(b_prev, "b_prev", n_out)
    Vs = out if out is not None else torch.empty_like(Vt)
    bs = torch.empty(n_out, dtype=torch.float32, device=Vt.device) if b_prev is not None else None
    ws = workspace
    if ws is None:
        nbytes = fold_mean_center_workspace_bytes(n_out, d_in)
        ws = torch.empty((nbytes + 15) // 16 * 2, dtype=torch.float64, device=Vt.device)
    _check(lib().flashnorm_fold_mean_center(_ptr(Vt), n_out, d_in, _dtype_code(Vt), _ptr(b_prev), _ptr(Vs),
                                            _ptr(bs), _ptr(ws), _stream(Vt)), "fold_mean_center")
    return Vs, bs


def linear(a, Wt_star, c_star=None, eps: float = 1e-5, mode: str = "rmsnorm", alpha: float = 0.5,
           path: str = "auto", out=None, workspace="auto"):
    """FlashNorm linear: z = (a W*) * rsqrt(mean(a^2) + eps) + c*  (PAPER.md:17, 177).

    a: [M, K]; Wt_star: [N, K] (same dtype, bf16 or f32); c_star: float32[N] or None.
    mode: rmsnorm | layernorm (input pre-centered via fold_mean_center) | dyt | none.
    workspace: "auto" allocates the scratch flashnorm_linear_workspace_bytes asks for
    (DyT on the GEMM path: tanh pre-pass, include/flashnorm.h); None forces the
    in-kernel tanh prologue; or a caller-owned CUDA tensor.
    """
    torch = _torch()
    _dev(a, "a")
    _dev(Wt_star, "Wt_star")
    if a.dim() != 2 or Wt_star.dim() != 2 or a.shape[1] != Wt_star.shape[1]:
        raise FlashNormError(2, "linear", f"a{list(a.shape)} and Wt_star{list(Wt_star.shape)}: need a[M,K], "
                                          "Wt_star[N,K]")
    if a.dtype != Wt_star.dtype:
        raise FlashNormError(3, "linear", f"a is {a.dtype} but Wt_star is {Wt_star.dtype}")
    M, K = a.shape
    N = Wt_star.shape[0]
    c_star = _vec(c_star, "c_star", N)
    z = out if out is not None else torch.empty((M, N), dtype=a.dtype, device=a.device)
    if isinstance(workspace, str):
        if workspace != "auto":
            raise FlashNormError(5, "linear", f"workspace must be 'auto', None or a CUDA tensor, got {workspace!r}")
        nb = linear_workspace_bytes(M, K, N, mode, a.dtype, path)
        workspace = torch.empty(nb, dtype=torch.uint8, device=a.device) if nb > 0 else None
    ws_bytes = 0
    if workspace is not None:
        _dev(workspace, "workspace")
        ws_bytes = workspace.numel() * workspace.element_size()
    st = lib().flashnorm_linear_ws(_ptr(a), _ptr(Wt_star), _ptr(c_star), M, K, N, float(eps), float(alpha),
                                   MODES[mode], _dtype_code(a), _ptr(z), PATHS[path], _ptr(workspace), ws_bytes,
                                   _stream(a))
    _check(st, "linear")
    return z


def linear_workspace_bytes(M: int, K: int, N: int, mode: str = "rmsnorm", dtype=None, path: str = "auto") -> int:
    """Scratch bytes flashnorm_linear_ws would use for this call (0 = none)."""
    torch = _torch()
    dt = _DT_F32 if dtype == torch.float32 else _DT_BF16
    return int(lib().flashnorm_linear_workspace_bytes(M, K, N, MODES[mode], dt, PATHS[path]))


def fold_glu_weights(Wg_t, Wu_t, g=None, out=None):
    """Gate/up folds for a GLU FFN: returns Wgu_star [2F, K], gate/up
    interleaved in 128-row blocks (include/flashnorm.h).  Wg_t, Wu_t: [F, K]."""
    torch = _torch()
    _dev(Wg_t, "Wg_t")
    _dev(Wu_t, "Wu_t")
    if Wg_t.shape != Wu_t.shape or Wg_t.dim() != 2 or Wg_t.dtype != Wu_t.dtype:
        raise FlashNormError(2, "fold_glu_weights", f"Wg_t{list(Wg_t.shape)} / Wu_t{list(Wu_t.shape)}: need two [F, K]")
    F, K = Wg_t.shape
    g = _vec(g, "g", K)
    W = out if out is not None else torch.empty((2 * F, K), dtype=Wg_t.dtype, device=Wg_t.device)
    _check(lib().flashnorm_fold_glu_weights(_ptr(Wg_t), _ptr(Wu_t), F, K, _dtype_code(Wg_t), _ptr(g), _ptr(W),
                                            _stream(Wg_t)), "fold_glu_weights")
    return W


def glu_linear(a, Wgu_star, eps: float = 1e-5, act: str = "silu", out=None, s_out=None):
    """Gate||up GEMM with the GLU epilogue: returns (h [M, F], s [M]) with y = (h W_down) * s
    (Figs 3(b)/4(b), readings c24-c25)."""
    torch = _torch()
    _dev(a, "a")
    _dev(Wgu_star, "Wgu_star")
    M, K = a.shape
    F = Wgu_star.shape[0] // 2
    h = out if out is not None else torch.empty((M, F), dtype=a.dtype, device=a.device)
    s = s_out if s_out is not None else torch.empty(M, dtype=torch.float32, device=a.device)
    _check(lib().flashnorm_glu_linear(_ptr(a), _ptr(Wgu_star), M, K, F, float(eps), GLU_ACTS[act], _dtype_code(a),
                                      _ptr(h), _ptr(s), _stream(a)), "glu_linear")
    return h, s


def qk_norm_rope_linear(a, Wt_star, n_q: int, n_k: int, head_dim: int, g_q, g_k, positions, cos_tab, sin_tab,
                        eps_qk: float = 1e-6, qk_scale: float = 1.0, eps: float = 1e-5, out=None):
    """[Q | K | V] with per-head QK-norm fused into RoPE (Figs 6(b)+7(b))."""
    torch = _torch()
    for t, nm in ((a, "a"), (Wt_star, "Wt_star"), (g_q, "g_q"), (g_k, "g_k"), (positions, "positions"),
                  (cos_tab, "cos_tab"), (sin_tab, "sin_tab")):
        _dev(t, nm)
    M, K = a.shape
    N = Wt_star.shape[0]
    z = out if out is not None else torch.empty((M, N), dtype=a.dtype, device=a.device)
    _check(lib().flashnorm_qk_norm_rope_linear(_ptr(a), _ptr(Wt_star), M, K, N, n_q, n_k, head_dim, _ptr(g_q),
                                               _ptr(g_k), float(eps_qk), _ptr(positions), _ptr(cos_tab),
                                               _ptr(sin_tab), float(qk_scale), float(eps), _dtype_code(a), _ptr(z),
                                               _stream(a)), "qk_norm_rope_linear")
    return z


def relu_ffn_up(a, Wt_star, eps: float = 1e-5, out=None, s_out=None):
    """Fig 2(b): h = relu(a W*_up) (unscaled), s = 1/RMSe(a); y = (h W_down) * s via linear_scaled."""
    torch = _torch()
    _dev(a, "a")
    _dev(Wt_star, "Wt_star")
    M, K = a.shape
    F = Wt_star.shape[0]
    h = out if out is not None else torch.empty((M, F), dtype=a.dtype, device=a.device)
    s = s_out if s_out is not None else torch.empty(M, dtype=torch.float32, device=a.device)
    _check(lib().flashnorm_relu_ffn_up(_ptr(a), _ptr(Wt_star), M, K, F, float(eps), _dtype_code(a), _ptr(h), _ptr(s),
                                       _stream(a)), "relu_ffn_up")
    return h, s


def linear_scaled(a, Wt_star, row_scale, c_star=None, out=None):
    """z = (a W*) * row_scale[m] + c*: the down projection with the deferred FFN-output scale."""
    torch = _torch()
    _dev(a, "a")
    _dev(Wt_star, "Wt_star")
    _dev(row_scale, "row_scale")
    M, K = a.shape
    N = Wt_star.shape[0]
    c_star = _vec(c_star, "c_star", N)
    z = out if out is not None else torch.empty((M, N), dtype=a.dtype, device=a.device)
    _check(lib().flashnorm_linear_scaled(_ptr(a), _ptr(Wt_star), _ptr(c_star), _ptr(row_scale), M, K, N,
                                         _dtype_code(a), _ptr(z), _stream(a)), "linear_scaled")
    return z


def fold_colsum(Wt_star, out=None):
    """u = 1^T W*: u[j] = sum_k W*t[j][k] (fp64 sum, one f32 rounding) — the correction vector of
    the deferred LayerNorm (NEXT-4, reading c29)."""
    torch = _torch()
    _dev(Wt_star, "Wt_star")
    N, K = Wt_star.shape
    u = out if out is not None else torch.empty(N, dtype=torch.float32, device=Wt_star.device)
    _check(lib().flashnorm_fold_colsum(_ptr(Wt_star), N, K, _dtype_code(Wt_star), _ptr(u), _stream(Wt_star)),
           "fold_colsum")
    return u


def layernorm_linear(a, Wt_star, u, c_star=None, eps: float = 1e-5, out=None):
    """LayerNorm -> linear with the mean AND the normalization deferred past the contraction:
    z = (a W* - mu u) / sqrt(var + eps) + c*, mu / var reduced beside the contraction (PAPER.md:33,
    42-46; reading c29).  W*, c* from fold_weights(W, g, b, c); u from fold_colsum(W*)."""
    torch = _torch()
    _dev(a, "a")
    _dev(Wt_star, "Wt_star")
    M, K = a.shape
    N = Wt_star.shape[0]
    u = _vec(u, "u", N)
    c_star = _vec(c_star, "c_star", N)
    z = out if out is not None else torch.empty((M, N), dtype=a.dtype, device=a.device)
    _check(lib().flashnorm_layernorm_linear(_ptr(a), _ptr(Wt_star), _ptr(u), _ptr(c_star), M, K, N, float(eps),
                                            _dtype_code(a), _ptr(z), _stream(a)), "layernorm_linear")
    return z


def linear_gather(a, Wt_star, dsts, col0: int, c_star=None, eps: float = 1e-5, mode: str = "rmsnorm",
                  alpha: float = 0.5):
    """This rank's column shard written by the GEMM epilogue into every buffer of `dsts` (each an
    [M, ldz] bf16 tensor: local, or peer-mapped gathered outputs) at columns [col0, col0 + N)."""
    _dev(a, "a")
    _dev(Wt_star, "Wt_star")
    M, K = a.shape
    N = Wt_star.shape[0]
    c_star = _vec(c_star, "c_star", N)
    if not dsts:
        raise FlashNormError(5, "linear_gather", "dsts is empty")
    ldz = dsts[0].shape[1]
    for d in dsts:
        _dev(d, "dst")
        if tuple(d.shape) != (M, ldz) or not d.is_contiguous() or d.dtype != a.dtype:
            raise FlashNormError(2, "linear_gather", f"every destination must be a contiguous [{M}, {ldz}] "
                                                    f"{a.dtype} tensor, got {d.dtype}{list(d.shape)}")
    ptrs = (ctypes.c_void_p * len(dsts))(*[d.data_ptr() for d in dsts])
    _check(lib().flashnorm_linear_gather(_ptr(a), _ptr(Wt_star), _ptr(c_star), M, K, N, float(eps), float(alpha),
                                         MODES[mode], _dtype_code(a), ptrs, len(dsts), ldz, int(col0), _stream(a)),
           "linear_gather")


def comm_unique_id() -> bytes:
    """An NCCL unique id (128 bytes) for flashnorm_comm_init; create on one rank, share it."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().flashnorm_comm_unique_id(buf), "comm_unique_id")
    return buf.raw


def comm_init(unique_id: bytes, nranks: int, rank: int) -> int:
    """NCCL communicator of this rank (call with this rank's GPU current); returns the handle."""
    if len(unique_id) != 128:
        raise FlashNormError(5, "comm_init", "unique_id must be 128 bytes")
    out = ctypes.c_void_p()
    _check(lib().flashnorm_comm_init(ctypes.create_string_buffer(unique_id, 128), int(nranks), int(rank),
                                     ctypes.byref(out)), "comm_init")
    return out.value


def comm_destroy(comm: int) -> None:
    _check(lib().flashnorm_comm_destroy(ctypes.c_void_p(comm)), "comm_destroy")


def allgather_columns(z_local, comm: int, nranks: int, out=None, workspace=None):
    """z [M, P*N_local] from every rank's column shard z_local [M, N_local] (NCCL all-gather through the
    C ABI, then the library's permute), on the current stream."""
    torch = _torch()
    _dev(z_local, "z_local")
    M, Nl = z_local.shape
    z = out if out is not None else torch.empty((M, nranks * Nl), dtype=z_local.dtype, device=z_local.device)
    if workspace is None:
        workspace = torch.empty((nranks, M, Nl), dtype=z_local.dtype, device=z_local.device)
    _check(lib().flashnorm_allgather_columns(_ptr(z_local), M, Nl, _dtype_code(z_local), _ptr(z), _ptr(workspace),
                                             ctypes.c_void_p(comm), _stream(z_local)), "allgather_columns")
    return z


def glu_ffn(a, Wgu_star, Wd_t, eps: float = 1e-5, act: str = "silu"):
    """The whole FlashNorm GLU FFN: two launches (gate||up with the GLU epilogue, then the down
    projection scaled at its output)."""
    h, s = glu_linear(a, Wgu_star, eps=eps, act=act)
    return linear_scaled(h, Wd_t, s)


def qkv_rope_linear(a, Wt_star, n_rope: int, head_dim: int, positions, cos_tab, sin_tab, qk_scale: float = 1.0,
                    eps: float = 1e-5, out=None):
    """[Q | K | V] = RoPE-fused FlashNorm projection (Fig 5(b)).
    positions: int32 [M]; cos_tab / sin_tab: float32 [max_pos, head_dim // 2]."""
    torch = _torch()
    _dev(a, "a")
    _dev(Wt_star, "Wt_star")
    for t, nm in ((positions, "positions"), (cos_tab, "cos_tab"), (sin_tab, "sin_tab")):
        _dev(t, nm)
    if positions.dtype != torch.int32 or cos_tab.dtype != torch.float32 or sin_tab.dtype != torch.float32:
        raise FlashNormError(3, "qkv_rope_linear", "positions must be int32, cos_tab / sin_tab float32")
    M, K = a.shape
    N = Wt_star.shape[0]
    z = out if out is not None else torch.empty((M, N), dtype=a.dtype, device=a.device)
    _check(lib().flashnorm_qkv_rope_linear(_ptr(a), _ptr(Wt_star), M, K, N, n_rope, head_dim, _ptr(positions),
                                           _ptr(cos_tab), _ptr(sin_tab), float(qk_scale), float(eps),
                                           _dtype_code(a), _ptr(z), _stream(a)), "qkv_rope_linear")
    return z


def linear_from_host(a_host, Wt_star, c_star, a_dev, z_dev, z_host, eps: float = 1e-5, mode: str = "rmsnorm",
                     alpha: float = 0.5, stream=None):
    """End-to-end call through the C ABI with HOST buffers (pinned a_host / z_host).

    Enqueues H2D(a) -> flashnorm_linear -> D2H(z) on the current stream (no sync).
    """
    torch = _torch()
    M, K = a_host.shape
    N = Wt_star.shape[0]
    st = stream if stream is not None else torch.cuda.current_stream(Wt_star.device)
    s = lib().flashnorm_linear_from_host(_ptr(a_host), _ptr(Wt_star), _ptr(c_star), M, K, N, float(eps),
                                         float(alpha), MODES[mode], _dtype_code(Wt_star), _ptr(a_dev), _ptr(z_dev),
                                         _ptr(z_host), ctypes.c_void_p(st.cuda_stream))
    _check(s, "linear_from_host")
    return z_host


def baseline_norm(a, g=None, b=None, eps: float = 1e-5, mode: str = "rmsnorm", alpha: float = 0.5, out=None):
    """Unfused normalization y = RN(Norm(a) * g + b) (measurement-only, Fig 1(a))."""
    torch = _torch()
    _dev(a, "a")
    M, K = a.shape
    g, b = _vec(g, "g", K), _vec(b, "b", K)
    y = out if out is not None else torch.empty_like(a)
    _check(lib().flashnorm_baseline_norm(_ptr(a), _ptr(g), _ptr(b), M, K, float(eps), MODES[mode], float(alpha),
                                         _dtype_code(a), _ptr(y), _stream(a)), "baseline_norm")
    return y


def gather_columns(z_parts, out=None):
    """z_parts [P, M, N_local] (all-gathered column shards) -> z [M, P*N_local]."""
    torch = _torch()
    _dev(z_parts, "z_parts")
    P, M, Nl = z_parts.shape
    z = out if out is not None else torch.empty((M, P * Nl), dtype=z_parts.dtype, device=z_parts.device)
    _check(lib().flashnorm_gather_columns(_ptr(z_parts), P, M, Nl, _dtype_code(z_parts), _ptr(z),
                                          _stream(z_parts)), "gather_columns")
    return z


def launch_count() -> int:
    return int(lib().flashnorm_launch_count())


def reset_launch_count() -> None:
    lib().flashnorm_reset_launch_count()


def version() -> str:
    return lib().flashnorm_version().decode()
