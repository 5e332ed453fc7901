"""paper_2407_09577_b200 — B200-native FlashNorm (arXiv 2407.09577) hot path.

Thin ctypes binding over ``libflashnorm.so`` (the C ABI in include/flashnorm.h); the
per-token entry (``linear`` → ``flashnorm_linear_ws``) goes through ``_pyfast``, a CPython
fast-call shim (csrc/pyfast.c) bound to the same library function.
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
    "fold_colsum", "layernorm_linear", "linear_gather", "linear_gather_multicast", "comm_unique_id", "comm_init",
    "comm_destroy",
    "allgather_columns", "comm_count",
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
    "flashnorm_linear_scaled_ws",
    "flashnorm_fold_colsum", "flashnorm_layernorm_linear", "flashnorm_linear_gather", "flashnorm_linear_gather_multicast",
    "flashnorm_comm_unique_id", "flashnorm_comm_init", "flashnorm_comm_destroy", "flashnorm_comm_count",
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
        "flashnorm_linear_scaled_ws": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _vp, _vp, _i64, _vp],
        "flashnorm_fold_colsum": [_vp, _i64, _i64, _int, _vp, _vp],
        "flashnorm_comm_unique_id": [_vp],
        "flashnorm_comm_init": [_vp, _int, _int, ctypes.POINTER(ctypes.c_void_p)],
        "flashnorm_comm_destroy": [_vp],
        "flashnorm_comm_count": [_vp, ctypes.POINTER(ctypes.c_int)],
        "flashnorm_allgather_workspace_bytes": [_i64, _i64, _i64, _int],
        "flashnorm_allgather_columns": [_vp, _i64, _i64, _int, _vp, _vp, _vp, _vp],
        "flashnorm_linear_gather": [_vp, _vp, _vp, _i64, _i64, _i64, _f32, _f32, _int, _int, _vp, _int, _i64, _i64,
                                    _vp],
        "flashnorm_layernorm_linear": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _f32, _int, _vp, _vp],
        "flashnorm_linear_gather_multicast": [_vp, _vp, _vp, _i64, _i64, _i64, _f32, _f32, _int, _int, _vp, _i64,
                                              _i64, _vp],
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
    global _FAST_LINEAR_WS
    try:  # the CPython fast-call shim (csrc/pyfast.c), bound to THIS library's function
        from . import _pyfast
        _pyfast.bind(ctypes.cast(L.flashnorm_linear_ws, ctypes.c_void_p).value)
        _FAST_LINEAR_WS = _pyfast.linear_ws
    except ImportError:
        _FAST_LINEAR_WS = L.flashnorm_linear_ws
    return L


_FAST_LINEAR_WS = None


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


def _mat(t, name: str, rows: Optional[int] = None, cols: Optional[int] = None, dtype=None):
    """A contiguous 2-D CUDA tensor, optionally of a given shape / dtype (the C side trusts the
    sizes it is given: a wrong shape here would read or write out of bounds on the GPU)."""
    _dev(t, name)
    if t.dim() != 2:
        raise FlashNormError(2, name, f"{name} must be 2-D, got {list(t.shape)}")
    if (rows is not None and t.shape[0] != rows) or (cols is not None and t.shape[1] != cols):
        want = f"[{'*' if rows is None else rows}, {'*' if cols is None else cols}]"
        raise FlashNormError(2, name, f"{name} must be {want}, got {list(t.shape)}")
    if dtype is not None and t.dtype != dtype:
        raise FlashNormError(3, name, f"{name} must be {dtype}, got {t.dtype}")
    return t


def _operands(a, Wt, name: str, w_name: str = "Wt_star"):
    """a [M, K] and W [N, K]: both CUDA, contiguous, 2-D, same dtype, same device, same K.
    Returns (M, K, N)."""
    _mat(a, "a")
    _mat(Wt, w_name)
    if a.shape[1] != Wt.shape[1]:
        raise FlashNormError(2, name, f"a{list(a.shape)} and {w_name}{list(Wt.shape)}: need a[M,K], {w_name}[N,K]")
    if a.dtype != Wt.dtype:
        raise FlashNormError(3, name, f"a is {a.dtype} but {w_name} is {Wt.dtype}")
    if a.device != Wt.device:
        raise FlashNormError(5, name, f"a is on {a.device} but {w_name} on {Wt.device}")
    _dtype_code(a)
    return a.shape[0], a.shape[1], Wt.shape[0]


def _out(t, name: str, shape, dtype, device):
    """A caller-supplied output buffer: exact shape, dtype and device, contiguous; else a new one."""
    torch = _torch()
    if t is None:
        return torch.empty(tuple(shape), dtype=dtype, device=device)
    _dev(t, name)
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != device:
        raise FlashNormError(2, name, f"{name} must be {dtype}{list(shape)} on {device}, "
                                      f"got {t.dtype}{list(t.shape)} on {t.device}")
    return t


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _raw_stream(device) -> int:
    """The current CUDA stream of `device` as an integer handle (torch's raw accessor: ~0.1 us
    against ~2 us for torch.cuda.current_stream(), which builds a Stream object)."""
    torch = _torch()
    get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if get is not None:
        return get(device.index if device.index is not None else torch.cuda.current_device())
    return torch.cuda.current_stream(device).cuda_stream


def _stream(t):
    return ctypes.c_void_p(_raw_stream(t.device))


# ------------------------------------------------------------------ public API

def fold_weights(Wt, g=None, b=None, c=None, out=None, c_out=None):
    """Fold norm weights g and norm bias b into (W*t, c*).  Wt: [N, K] (nn.Linear layout).

    PAPER.md:25 (c* = c + b W, original W) then PAPER.md:16 (W*_ij = g_i W_ij).
    Returns (Wt_star [N, K] same dtype, c_star float32[N] or None).
    """
    torch = _torch()
    _mat(Wt, "Wt")
    _dtype_code(Wt)
    N, K = Wt.shape
    g, b, c = _vec(g, "g", K), _vec(b, "b", K), _vec(c, "c", N)
    Ws = _out(out, "out", (N, K), Wt.dtype, Wt.device)
    cs = None
    if c_out is not None or b is not None or c is not None:
        cs = _out(c_out, "c_out", (N,), torch.float32, Wt.device)
    _check(lib().flashnorm_fold_weights(_ptr(Wt), N, K, _dtype_code(Wt), _ptr(g), _ptr(b), _ptr(c), _ptr(Ws),
                                        _ptr(cs), _stream(Wt)), "fold_weights")
    return Ws, cs


def fold_mean_center_workspace_bytes(n_out: int, d_in: int) -> int:
    """Bytes of device scratch flashnorm_fold_mean_center uses (fp64 partial column sums + s_i / n)."""
    return int(lib().flashnorm_fold_mean_center_workspace_bytes(n_out, d_in))


def fold_mean_center(Vt, b_prev=None, out=None, workspace=None):
    """Fold LayerNorm's mean centering into the preceding layer.  Vt: [n_out, d_in].

    PAPER.md:42-49: v*_ij = v_ij - s_i/n; b_prev* = b_prev - mean(b_prev) (reading c7).
    Returns (Vt_star, b_prev_star or None).
    """
    torch = _torch()
    _mat(Vt, "Vt")
    _dtype_code(Vt)
    n_out, d_in = Vt.shape
    b_prev = _vec(b_prev, "b_prev", n_out)
    Vs = _out(out, "out", (n_out, d_in), Vt.dtype, Vt.device)
    bs = torch.empty(n_out, dtype=torch.float32, device=Vt.device) if b_prev is not None else None
    ws = workspace
    nbytes = fold_mean_center_workspace_bytes(n_out, d_in)
    if ws is None:
        ws = torch.empty((nbytes + 15) // 16 * 2, dtype=torch.float64, device=Vt.device)
    else:
        _dev(ws, "workspace")
        if ws.numel() * ws.element_size() < nbytes:
            raise FlashNormError(2, "fold_mean_center", f"workspace holds {ws.numel() * ws.element_size()} bytes, "
                                                        f"needs {nbytes}")
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
    M, K, N = _operands(a, Wt_star, "linear")
    if mode not in MODES or path not in PATHS:
        raise FlashNormError(5, "linear", f"mode {mode!r} / path {path!r}: mode in {list(MODES)}, path in {list(PATHS)}")
    c_star = _vec(c_star, "c_star", N)
    dev = a.device
    z = _out(out, "out", (M, N), a.dtype, dev)
    stream = _raw_stream(dev)
    if isinstance(workspace, str):
        if workspace != "auto":
            raise FlashNormError(5, "linear", f"workspace must be 'auto', None or a CUDA tensor, got {workspace!r}")
        key = (M, K, N, mode, a.dtype, path)
        nb = _WSB_CACHE.get(key)
        if nb is None:
            nb = _WSB_CACHE[key] = linear_workspace_bytes(M, K, N, mode, a.dtype, path)
        workspace = _auto_workspace(nb, dev, stream) if nb > 0 else None
    ws_bytes = 0
    if workspace is not None:
        _dev(workspace, "workspace")
        ws_bytes = workspace.numel() * workspace.element_size()
    # raw integer pointers (ctypes converts them for the c_void_p argtypes): the decode path is
    # host-bound when launched eagerly, so this wrapper keeps its per-call work small
    if _FAST_LINEAR_WS is None:
        lib()
    st = _FAST_LINEAR_WS(a.data_ptr(), Wt_star.data_ptr(), None if c_star is None else c_star.data_ptr(),
                                   M, K, N, eps, alpha, MODES[mode], _DT_F32 if a.dtype == torch.float32 else _DT_BF16,
                                   z.data_ptr(), PATHS[path], None if workspace is None else workspace.data_ptr(),
                                   ws_bytes, stream)
    if st:
        _check(st, "linear")
    return z


_WSB_CACHE = {}  # (M, K, N, mode, dtype, path) -> flashnorm_linear_workspace_bytes
_WS_CACHE = {}


def _auto_workspace(nbytes: int, device, stream=None):
    """The library-facing scratch of linear(workspace="auto"): one zero-filled buffer per (device,
    stream), grown on demand and reused — its first 4 KiB (stream-K flags) must be zero before a
    call and every call leaves them zero (include/flashnorm.h flashnorm_linear_ws)."""
    torch = _torch()
    key = (device.index, _raw_stream(device) if stream is None else stream)
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf


def linear_workspace_bytes(M: int, K: int, N: int, mode: str = "rmsnorm", dtype=None, path: str = "auto") -> int:
    """Scratch bytes flashnorm_linear_ws would use for this call (0 = none)."""
    torch = _torch()
    dt = _DT_F32 if dtype == torch.float32 else _DT_BF16
    return int(lib().flashnorm_linear_workspace_bytes(M, K, N, MODES[mode], dt, PATHS[path]))


def fold_glu_weights(Wg_t, Wu_t, g=None, out=None):
    """Gate/up folds for a GLU FFN: returns Wgu_star [2F, K], gate/up
    interleaved in 128-row blocks (include/flashnorm.h).  Wg_t, Wu_t: [F, K]."""
    _mat(Wg_t, "Wg_t")
    _mat(Wu_t, "Wu_t")
    _dtype_code(Wg_t)
    if Wg_t.shape != Wu_t.shape or Wg_t.dtype != Wu_t.dtype or Wg_t.device != Wu_t.device:
        raise FlashNormError(2, "fold_glu_weights", f"Wg_t{list(Wg_t.shape)} / Wu_t{list(Wu_t.shape)}: need two [F, K]")
    F, K = Wg_t.shape
    g = _vec(g, "g", K)
    W = _out(out, "out", (2 * F, K), Wg_t.dtype, Wg_t.device)
    _check(lib().flashnorm_fold_glu_weights(_ptr(Wg_t), _ptr(Wu_t), F, K, _dtype_code(Wg_t), _ptr(g), _ptr(W),
                                            _stream(Wg_t)), "fold_glu_weights")
    return W


def glu_linear(a, Wgu_star, eps: float = 1e-5, act: str = "silu", out=None, s_out=None):
    """Gate||up GEMM with the GLU epilogue: returns (h [M, F], s [M]) with y = (h W_down) * s
    (Figs 3(b)/4(b), readings c24-c25)."""
    torch = _torch()
    M, K, N2 = _operands(a, Wgu_star, "glu_linear", "Wgu_star")
    if N2 % 2 or act not in GLU_ACTS:
        raise FlashNormError(2, "glu_linear", f"Wgu_star must be [2F, K] (got {N2} rows), act in {list(GLU_ACTS)}")
    F = N2 // 2
    h = _out(out, "out", (M, F), a.dtype, a.device)
    s = _out(s_out, "s_out", (M,), torch.float32, a.device)
    _check(lib().flashnorm_glu_linear(_ptr(a), _ptr(Wgu_star), M, K, F, float(eps), GLU_ACTS[act], _dtype_code(a),
                                      _ptr(h), _ptr(s), _stream(a)), "glu_linear")
    return h, s


def qk_norm_rope_linear(a, Wt_star, n_q: int, n_k: int, head_dim: int, g_q, g_k, positions, cos_tab, sin_tab,
                        eps_qk: float = 1e-6, qk_scale: float = 1.0, eps: float = 1e-5, out=None):
    """[Q | K | V] with per-head QK-norm fused into RoPE (Figs 6(b)+7(b))."""
    M, K, N = _operands(a, Wt_star, "qk_norm_rope_linear")
    g_q, g_k = _vec(g_q, "g_q", head_dim), _vec(g_k, "g_k", head_dim)
    _rope_tables(positions, cos_tab, sin_tab, M, head_dim, "qk_norm_rope_linear")
    z = _out(out, "out", (M, N), a.dtype, a.device)
    _check(lib().flashnorm_qk_norm_rope_linear(_ptr(a), _ptr(Wt_star), M, K, N, n_q, n_k, head_dim, _ptr(g_q),
                                               _ptr(g_k), float(eps_qk), _ptr(positions), _ptr(cos_tab),
                                               _ptr(sin_tab), float(qk_scale), float(eps), _dtype_code(a), _ptr(z),
                                               _stream(a)), "qk_norm_rope_linear")
    return z


def relu_ffn_up(a, Wt_star, eps: float = 1e-5, out=None, s_out=None):
    """Fig 2(b): h = relu(a W*_up) (unscaled), s = 1/RMSe(a); y = (h W_down) * s via linear_scaled."""
    torch = _torch()
    M, K, F = _operands(a, Wt_star, "relu_ffn_up")
    h = _out(out, "out", (M, F), a.dtype, a.device)
    s = _out(s_out, "s_out", (M,), torch.float32, a.device)
    _check(lib().flashnorm_relu_ffn_up(_ptr(a), _ptr(Wt_star), M, K, F, float(eps), _dtype_code(a), _ptr(h), _ptr(s),
                                       _stream(a)), "relu_ffn_up")
    return h, s


def linear_scaled(a, Wt_star, row_scale, c_star=None, out=None, workspace="auto"):
    """z = (a W*) * row_scale[m] + c*: the down projection with the deferred FFN-output scale.
    workspace: "auto" (the stream-K scratch flashnorm_linear_workspace_bytes asks for, if any),
    None, or a caller-owned CUDA tensor (flashnorm_linear_scaled_ws)."""
    M, K, N = _operands(a, Wt_star, "linear_scaled")
    row_scale = _vec(row_scale, "row_scale", M)
    c_star = _vec(c_star, "c_star", N)
    z = _out(out, "out", (M, N), a.dtype, a.device)
    if isinstance(workspace, str):
        if workspace != "auto":
            raise FlashNormError(5, "linear_scaled", f"workspace must be 'auto', None or a CUDA tensor, got {workspace!r}")
        nb = linear_workspace_bytes(M, K, N, "none", a.dtype, "auto")
        workspace = _auto_workspace(nb, a.device) if nb > 0 else None
    ws_bytes = 0
    if workspace is not None:
        _dev(workspace, "workspace")
        ws_bytes = workspace.numel() * workspace.element_size()
    _check(lib().flashnorm_linear_scaled_ws(_ptr(a), _ptr(Wt_star), _ptr(c_star), _ptr(row_scale), M, K, N,
                                            _dtype_code(a), _ptr(z), _ptr(workspace), ws_bytes, _stream(a)),
           "linear_scaled")
    return z


def fold_colsum(Wt_star, out=None):
    """u = 1^T W*: u[j] = sum_k W*t[j][k] (fp64 sum, one f32 rounding) — the correction vector of
    the deferred LayerNorm (NEXT-4, reading c29)."""
    torch = _torch()
    _mat(Wt_star, "Wt_star")
    _dtype_code(Wt_star)
    N, K = Wt_star.shape
    u = _out(out, "out", (N,), torch.float32, Wt_star.device)
    _check(lib().flashnorm_fold_colsum(_ptr(Wt_star), N, K, _dtype_code(Wt_star), _ptr(u), _stream(Wt_star)),
           "fold_colsum")
    return u


def layernorm_linear(a, Wt_star, u, c_star=None, eps: float = 1e-5, out=None):
    """LayerNorm -> linear with the mean AND the normalization deferred past the contraction:
    z = (a W* - mu u) / sqrt(var + eps) + c*, mu / var reduced beside the contraction (PAPER.md:33,
    42-46; reading c29).  W*, c* from fold_weights(W, g, b, c); u from fold_colsum(W*)."""
    M, K, N = _operands(a, Wt_star, "layernorm_linear")
    u = _vec(u, "u", N)
    c_star = _vec(c_star, "c_star", N)
    z = _out(out, "out", (M, N), a.dtype, a.device)
    _check(lib().flashnorm_layernorm_linear(_ptr(a), _ptr(Wt_star), _ptr(u), _ptr(c_star), M, K, N, float(eps),
                                            _dtype_code(a), _ptr(z), _stream(a)), "layernorm_linear")
    return z


def linear_gather(a, Wt_star, dsts, col0: int, c_star=None, eps: float = 1e-5, mode: str = "rmsnorm",
                  alpha: float = 0.5):
    """This rank's column shard written by the GEMM epilogue into every buffer of `dsts` (each an
    [M, ldz] bf16 tensor: local, or peer-mapped gathered outputs) at columns [col0, col0 + N)."""
    M, K, N = _operands(a, Wt_star, "linear_gather")
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


def linear_gather_multicast(a, Wt_star, z_mc: int, ldz: int, col0: int, c_star=None, eps: float = 1e-5,
                            mode: str = "rmsnorm", alpha: float = 0.5):
    """This rank's column shard stored by the GEMM epilogue through an NVLS multicast address `z_mc`
    (an integer device address, e.g. torch symmetric memory's multicast_ptr): the NVSwitch writes it
    into every rank's [M, ldz] buffer at columns [col0, col0 + N) (include/flashnorm.h)."""
    M, K, N = _operands(a, Wt_star, "linear_gather_multicast")
    c_star = _vec(c_star, "c_star", N)
    _check(lib().flashnorm_linear_gather_multicast(_ptr(a), _ptr(Wt_star), _ptr(c_star), M, K, N, float(eps),
                                                   float(alpha), MODES[mode], _dtype_code(a), ctypes.c_void_p(z_mc),
                                                   int(ldz), int(col0), _stream(a)), "linear_gather_multicast")


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


def comm_count(comm: int) -> int:
    """Number of ranks of a communicator from comm_init (ncclCommCount)."""
    n = ctypes.c_int(0)
    _check(lib().flashnorm_comm_count(ctypes.c_void_p(comm), ctypes.byref(n)), "comm_count")
    return int(n.value)


def allgather_columns(z_local, comm: int, nranks: Optional[int] = None, out=None, workspace=None):
    """z [M, P*N_local] from every rank's column shard z_local [M, N_local] (NCCL all-gather through the
    C ABI, then the library's permute), on the current stream.  P is the communicator's rank count
    (a given `nranks` must equal it); out / workspace are checked against it."""
    _mat(z_local, "z_local")
    _dtype_code(z_local)
    P = comm_count(comm)
    if nranks is not None and int(nranks) != P:
        raise FlashNormError(5, "allgather_columns", f"nranks={nranks} but the communicator has {P} ranks")
    M, Nl = z_local.shape
    z = _out(out, "out", (M, P * Nl), z_local.dtype, z_local.device)
    if workspace is None:
        workspace = _torch().empty((P, M, Nl), dtype=z_local.dtype, device=z_local.device)
    else:
        _dev(workspace, "workspace")
        if workspace.numel() * workspace.element_size() < P * M * Nl * z_local.element_size():
            raise FlashNormError(2, "allgather_columns", f"workspace must hold {P}*{M}*{Nl} elements")
    _check(lib().flashnorm_allgather_columns(_ptr(z_local), M, Nl, _dtype_code(z_local), _ptr(z), _ptr(workspace),
                                             ctypes.c_void_p(comm), _stream(z_local)), "allgather_columns")
    return z


def glu_ffn(a, Wgu_star, Wd_t, eps: float = 1e-5, act: str = "silu"):
    """The whole FlashNorm GLU FFN: two launches (gate||up with the GLU epilogue, then the down
    projection scaled at its output)."""
    h, s = glu_linear(a, Wgu_star, eps=eps, act=act)
    return linear_scaled(h, Wd_t, s)


def _rope_tables(positions, cos_tab, sin_tab, M: int, head_dim: int, name: str):
    """positions int32[M]; cos_tab / sin_tab float32[max_pos, head_dim // 2] (reading c26).  Positions
    must lie in [0, max_pos): the kernels index the tables with them (checked here on the device
    tensor with one small D2H read — skipped while the stream is being captured into a CUDA graph,
    where a sync is illegal; the caller then owns the range)."""
    torch = _torch()
    if head_dim <= 0 or head_dim % 2:
        raise FlashNormError(5, name, f"head_dim = {head_dim} must be positive and even (RoPE pairs)")
    _dev(positions, "positions")
    if positions.dtype != torch.int32 or positions.dim() != 1 or positions.shape[0] != M:
        raise FlashNormError(3, name, f"positions must be int32[{M}], got {positions.dtype}{list(positions.shape)}")
    _mat(cos_tab, "cos_tab", cols=head_dim // 2, dtype=torch.float32)
    _mat(sin_tab, "sin_tab", rows=cos_tab.shape[0], cols=head_dim // 2, dtype=torch.float32)
    if M > 0 and not torch.cuda.is_current_stream_capturing():
        lo, hi = (int(v) for v in torch.aminmax(positions))
        if lo < 0 or hi >= cos_tab.shape[0]:
            raise FlashNormError(5, name, f"positions span [{lo}, {hi}] outside the {cos_tab.shape[0]}-row tables")


def qkv_rope_linear(a, Wt_star, n_rope: int, head_dim: int, positions, cos_tab, sin_tab, qk_scale: float = 1.0,
                    eps: float = 1e-5, out=None):
    """[Q | K | V] = RoPE-fused FlashNorm projection (Fig 5(b)).
    positions: int32 [M]; cos_tab / sin_tab: float32 [max_pos, head_dim // 2]."""
    M, K, N = _operands(a, Wt_star, "qkv_rope_linear")
    _rope_tables(positions, cos_tab, sin_tab, M, head_dim, "qkv_rope_linear")
    z = _out(out, "out", (M, N), a.dtype, a.device)
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
    _mat(Wt_star, "Wt_star")
    if a_host.is_cuda or z_host.is_cuda or a_host.dim() != 2 or not (a_host.is_contiguous() and z_host.is_contiguous()):
        raise FlashNormError(2, "linear_from_host", "a_host / z_host must be contiguous 2-D host tensors")
    M, K = a_host.shape
    N = Wt_star.shape[0]
    if K != Wt_star.shape[1] or a_host.dtype != Wt_star.dtype:
        raise FlashNormError(2, "linear_from_host", f"a_host {a_host.dtype}{list(a_host.shape)} vs Wt_star "
                                                    f"{Wt_star.dtype}{list(Wt_star.shape)}")
    if tuple(z_host.shape) != (M, N) or z_host.dtype != a_host.dtype:
        raise FlashNormError(2, "linear_from_host", f"z_host must be {a_host.dtype}[{M}, {N}]")
    _out(a_dev, "a_dev", (M, K), a_host.dtype, Wt_star.device)
    _out(z_dev, "z_dev", (M, N), a_host.dtype, Wt_star.device)
    c_star = _vec(c_star, "c_star", N)
    st = stream if stream is not None else torch.cuda.current_stream(Wt_star.device)
    s = lib().flashnorm_linear_from_host(_ptr(a_host), _ptr(Wt_star), _ptr(c_star), M, K, N, float(eps),
                                         float(alpha), MODES[mode], _dtype_code(Wt_star), _ptr(a_dev), _ptr(z_dev),
                                         _ptr(z_host), ctypes.c_void_p(st.cuda_stream))
    _check(s, "linear_from_host")
    return z_host


def baseline_norm(a, g=None, b=None, eps: float = 1e-5, mode: str = "rmsnorm", alpha: float = 0.5, out=None):
    """Unfused normalization y = RN(Norm(a) * g + b) (measurement-only, Fig 1(a))."""
    _mat(a, "a")
    _dtype_code(a)
    M, K = a.shape
    g, b = _vec(g, "g", K), _vec(b, "b", K)
    y = _out(out, "out", (M, K), a.dtype, a.device)
    _check(lib().flashnorm_baseline_norm(_ptr(a), _ptr(g), _ptr(b), M, K, float(eps), MODES[mode], float(alpha),
                                         _dtype_code(a), _ptr(y), _stream(a)), "baseline_norm")
    return y


def gather_columns(z_parts, out=None):
    """z_parts [P, M, N_local] (all-gathered column shards) -> z [M, P*N_local]."""
    _dev(z_parts, "z_parts")
    _dtype_code(z_parts)
    if z_parts.dim() != 3:
        raise FlashNormError(2, "gather_columns", f"z_parts must be [P, M, N_local], got {list(z_parts.shape)}")
    P, M, Nl = z_parts.shape
    z = _out(out, "out", (M, P * Nl), z_parts.dtype, z_parts.device)
    _check(lib().flashnorm_gather_columns(_ptr(z_parts), P, M, Nl, _dtype_code(z_parts), _ptr(z),
                                          _stream(z_parts)), "gather_columns")
    return z


def launch_count() -> int:
    return int(lib().flashnorm_launch_count())


def reset_launch_count() -> None:
    lib().flashnorm_reset_launch_count()


def version() -> str:
    return lib().flashnorm_version().decode()
