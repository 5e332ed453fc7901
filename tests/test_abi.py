"""The C-ABI library loads and exports every symbol include/flashnorm.h declares;
host-side validation returns the documented status codes (no GPU needed: every
check below fails before any CUDA call)."""
import ctypes
import os
import re

import pytest

import paper_2407_09577_b200 as fn
from paper_2407_09577_b200 import build as fnbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    fnbuild.build()
    return fn.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "flashnorm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(flashnorm_\w+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(fn.EXPORTS)


def test_every_declared_symbol_is_exported(L):
    for name in declared_symbols():
        assert hasattr(L, name), name
    # and by the dynamic symbol table (extern "C", unmangled)
    out = os.popen(f"nm -D --defined-only {fn.lib_path}").read()
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {fn.lib_path} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


def test_version_and_status_strings(L):
    assert "sm_100a" in fn.version()
    assert L.flashnorm_status_string(0) == b"FN_OK"
    assert L.flashnorm_status_string(4) == b"FN_ERR_ALIGN"
    assert L.flashnorm_status_string(99) == b"FN_ERR_UNKNOWN"


def test_workspace_size(L):
    # 32-row fp64 partial column sums + s_i / n (include/flashnorm.h fold_mean_center numerics)
    assert fn.fold_mean_center_workspace_bytes(4096, 4096) == (128 + 1) * 4096 * 8
    assert fn.fold_mean_center_workspace_bytes(33, 16) == (2 + 1) * 16 * 8
    assert fn.fold_mean_center_workspace_bytes(0, 16) == 0


P = ctypes.c_void_p


def _lin(L, a=0x1000, w=0x2000, c=None, M=4, K=64, N=64, eps=1e-5, alpha=0.5, mode=0, dt=0, z=0x3000, path=0):
    return L.flashnorm_linear_ex(P(a), P(w), P(c), M, K, N, eps, alpha, mode, dt, P(z), path, None)


def test_linear_validation_codes(L):
    assert _lin(L, a=None) == 1                                     # FN_ERR_NULL
    assert _lin(L, K=0) == 2                                        # FN_ERR_SHAPE
    assert _lin(L, M=-1) == 2
    assert _lin(L, dt=7) == 3                                       # FN_ERR_DTYPE
    assert _lin(L, K=60) == 4                                       # FN_ERR_ALIGN (bf16 needs K % 8)
    assert b"K = 60" in L.flashnorm_last_error()
    assert _lin(L, N=12) == 4
    assert _lin(L, a=0x1008) == 4                                   # misaligned pointer
    assert _lin(L, eps=-1.0) == 5                                   # FN_ERR_VALUE
    assert _lin(L, eps=float("nan")) == 5
    assert _lin(L, mode=2, alpha=float("inf")) == 5
    assert _lin(L, mode=9) == 5
    assert _lin(L, z=0x1000) == 5                                   # aliasing
    assert _lin(L, dt=1, path=1) == 6                               # FN_ERR_UNSUPPORTED: f32 on tcgen05
    assert _lin(L, M=17, path=2) == 6                               # decode path is M <= 16
    assert _lin(L, M=0) == 0                                        # empty batch: no-op


def test_linear_ws_validation_codes(L):
    f = L.flashnorm_linear_ws
    args = (P(0x1000), P(0x2000), None, 300, 64, 64, 1e-5, 0.5, 2, 0, P(0x3000), 0)
    assert f(*args, None, 16, None) == 1                              # bytes without a pointer
    assert f(*args, P(0x4008), 300 * 64 * 2, None) == 4               # misaligned workspace
    assert f(*args, P(0x3000), 300 * 64 * 2, None) == 5               # aliases z
    assert f(*args, P(0x4000), 300 * 64 * 2 - 16, None) == 5          # too small for the DyT pre-pass
    assert f(*args[:11], 9, P(0x4000), 0, None) == 5                  # unknown path
    wb = L.flashnorm_linear_workspace_bytes
    assert wb(300, 64, 64, 2, 0, 0) == 4096 + 300 * 64 * 2            # DyT GEMM: 4 KiB flags + M*K*2
    assert wb(8, 64, 64, 2, 0, 0) == 0                                # DyT decode: none
    assert wb(300, 64, 64, 0, 0, 0) == 0                              # rmsnorm: none
    assert wb(300, 64, 64, 2, 1, 0) == 0                              # f32: none


def test_pyfast_shim_is_bound_and_returns_the_c_status(L):
    """linear() calls flashnorm_linear_ws through the CPython fast-call shim (csrc/pyfast.c) bound
    to this library's function: the same status codes as the ctypes call, same thread-local error."""
    import importlib
    fast = importlib.import_module("paper_2407_09577_b200._pyfast")
    assert fn._FAST_LINEAR_WS is fast.linear_ws
    args = (0x1000, 0x2000, None, 300, 64, 64, 1e-5, 0.5, 2, 0, 0x3000, 0)
    assert fast.linear_ws(*args, None, 16, None) == 1                 # bytes without a pointer
    assert b"workspace" in L.flashnorm_last_error()
    assert fast.linear_ws(*args, 0x4008, 300 * 64 * 2, None) == 4     # misaligned workspace
    assert fast.linear_ws(*args[:11], 9, 0x4000, 0, None) == 5        # unknown path
    assert fast.linear_ws(None, None, None, 1, 64, 64, 1e-5, 0.5, 0, 0, None, 0, None, 0, None) == 1
    with pytest.raises(TypeError):
        fast.linear_ws(*args)


def test_linear_scaled_ws_validation_codes(L):
    f = L.flashnorm_linear_scaled_ws
    args = (P(0x1000), P(0x2000), None, P(0x5000), 300, 64, 64, 0, P(0x3000))
    assert f(*args[:3], None, *args[4:], None, 0, None) == 1          # row_scale NULL
    assert f(*args[:3], P(0x5008), *args[4:], None, 0, None) == 4     # misaligned row_scale
    assert f(*args, None, 16, None) == 1                              # bytes without a pointer
    assert f(*args, P(0x4008), 4096, None) == 4                       # misaligned workspace
    assert f(*args, P(0x3000), 4096, None) == 5                       # aliases z
    assert f(*args[:7], 1, *args[8:], None, 0, None) == 6             # f32: bf16-only entry
    wb = L.flashnorm_linear_workspace_bytes
    assert wb(4096, 14336, 4096, 3, 0, 0) > 4096                      # mode none, K >= 8192: stream-K scratch
    assert wb(2048, 4096, 4096, 3, 0, 0) == 0                         # K = 4096: whole tiles


def test_glu_validation_codes(L):
    gl = L.flashnorm_glu_linear
    assert gl(P(0x1000), P(0x2000), 4, 64, 100, 1e-5, 0, 0, P(0x3000), P(0x4000), None) == 2   # F % 128
    assert gl(P(0x1000), P(0x2000), 4, 64, 128, 1e-5, 7, 0, P(0x3000), P(0x4000), None) == 5   # act
    assert gl(P(0x1000), P(0x2000), 4, 64, 128, 1e-5, 0, 1, P(0x3000), P(0x4000), None) == 6   # f32
    assert gl(P(0x1000), P(0x2000), 4, 64, 128, 1e-5, 0, 0, P(0x3000), None, None) == 1        # s
    assert gl(P(0x1000), P(0x2000), 4, 64, 128, 1e-5, 0, 0, P(0x1000), P(0x4000), None) == 5   # h aliases a
    fg = L.flashnorm_fold_glu_weights
    assert fg(P(0x1000), P(0x2000), 100, 64, 0, None, P(0x3000), None) == 2                    # F % 128
    assert fg(P(0x1000), P(0x2000), 128, 60, 0, None, P(0x3000), None) == 4                    # K % 8
    assert fg(P(0x1000), P(0x2000), 128, 64, 0, None, P(0x1000), None) == 5                    # aliasing
    ls = L.flashnorm_linear_scaled
    assert ls(P(0x1000), P(0x2000), None, None, 4, 64, 64, 0, P(0x3000), None) == 1            # no scale
    assert ls(P(0x1000), P(0x2000), None, P(0x4000), 4, 64, 64, 1, P(0x3000), None) == 6       # f32


def test_fold_validation_codes(L):
    f = L.flashnorm_fold_weights
    assert f(P(0x1000), 8, 64, 0, None, P(0x4000), None, P(0x2000), None, None) == 1   # b without c_star
    assert f(P(0x1000), 0, 64, 0, None, None, None, P(0x2000), None, None) == 2
    assert f(P(0x1000), 8, 63, 1, None, None, None, P(0x2000), None, None) == 4
    assert f(P(0x1000), 8, 64, 0, None, None, None, P(0x1000), None, None) == 5       # aliasing
    g = L.flashnorm_fold_mean_center
    assert g(P(0x1000), 8, 64, 0, P(0x5000), P(0x2000), None, P(0x3000), None) == 1   # b_prev without output
    assert g(P(0x1000), 8, 64, 0, None, P(0x2000), None, None, None) == 1             # no workspace
    assert g(P(0x1000), 8, 12, 0, None, P(0x2000), None, P(0x3000), None) == 4


def test_layernorm_exact_validation_codes(L):
    cs = L.flashnorm_fold_colsum
    assert cs(P(0x1000), 8, 64, 0, None, None) == 1                                   # no u
    assert cs(P(0x1000), 0, 64, 0, P(0x2000), None) == 2
    assert cs(P(0x1000), 8, 60, 0, P(0x2000), None) == 4                              # K % 8
    assert cs(P(0x1000), 8, 64, 5, P(0x2000), None) == 3                              # dtype
    ln = L.flashnorm_layernorm_linear
    assert ln(P(0x1000), P(0x2000), None, None, 4, 64, 64, 1e-5, 0, P(0x3000), None) == 1   # no u
    assert ln(P(0x1000), P(0x2000), P(0x4000), None, 4, 60, 64, 1e-5, 0, P(0x3000), None) == 4
    assert ln(P(0x1000), P(0x2000), P(0x4000), None, 4, 64, 64, -1.0, 0, P(0x3000), None) == 5  # eps < 0
    assert ln(P(0x1000), P(0x2000), P(0x4004), None, 4, 64, 64, 1e-5, 0, P(0x3000), None) == 4  # u align
    assert ln(P(0x1000), P(0x2000), P(0x4000), None, 0, 64, 64, 1e-5, 0, P(0x3000), None) == 0  # M = 0


def test_python_binding_refuses_cpu_tensors():
    import torch
    a = torch.zeros(4, 64, dtype=torch.bfloat16)
    w = torch.zeros(64, 64, dtype=torch.bfloat16)
    with pytest.raises(fn.FlashNormError, match="CUDA tensor"):
        fn.linear(a, w)
    with pytest.raises(fn.FlashNormError, match="CUDA tensor"):
        fn.fold_weights(w)


def test_linear_gather_validation_codes(L):
    import ctypes
    f = L.flashnorm_linear_gather
    one = (ctypes.c_void_p * 1)(0x3000)
    assert f(P(0x1000), P(0x2000), None, 4, 64, 64, 1e-5, 0.5, 0, 1, one, 1, 64, 0, None) == 6     # f32
    assert f(P(0x1000), P(0x2000), None, 4, 64, 64, 1e-5, 0.5, 0, 0, one, 0, 64, 0, None) == 5     # ndst
    assert f(P(0x1000), P(0x2000), None, 4, 64, 64, 1e-5, 0.5, 0, 0, None, 1, 64, 0, None) == 1    # dsts
    assert f(P(0x1000), P(0x2000), None, 4, 64, 64, 1e-5, 0.5, 0, 0, one, 1, 96, 40, None) == 2    # ldz
    assert f(P(0x1000), P(0x2000), None, 4, 64, 64, 1e-5, 0.5, 0, 0, one, 1, 132, 68, None) == 4   # col0 % 8
    bad = (ctypes.c_void_p * 1)(0x3004)
    assert f(P(0x1000), P(0x2000), None, 4, 64, 64, 1e-5, 0.5, 0, 0, bad, 1, 64, 0, None) == 4     # align


def test_nccl_entry_validation_codes(L):
    assert L.flashnorm_status_string(8) == b"FN_ERR_NCCL"
    assert L.flashnorm_comm_unique_id(None) == 1
    assert L.flashnorm_comm_init(None, 1, 0, None) == 1
    assert L.flashnorm_comm_init(P(0x1000), 2, 2, None) in (1, 5)
    assert L.flashnorm_comm_destroy(None) == 0
    assert L.flashnorm_allgather_workspace_bytes(4, 8, 64, 0) == 4 * 8 * 64 * 2
    f = L.flashnorm_allgather_columns
    assert f(P(0x1000), 8, 64, 0, P(0x2000), P(0x3000), None, None) == 1        # comm
    assert f(P(0x1000), 8, 0, 0, P(0x2000), P(0x3000), P(0x4000), None) == 2    # N_local
    assert f(P(0x1000), 8, 64, 7, P(0x2000), P(0x3000), P(0x4000), None) == 3   # dtype
    assert f(P(0x1000), 8, 64, 0, P(0x2000), P(0x2000), P(0x4000), None) == 5   # workspace aliases z
