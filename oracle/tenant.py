"""ORACLE / TEST INFRASTRUCTURE ONLY — numpy/ctypes view of oracle/_build/libtenant_ref.so,
the plain-C restatement of the tenant-kernel math (oracle/tenant_ref.c)."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_LIB = Path(__file__).resolve().parent / "_build" / "libtenant_ref.so"
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB.exists():
            raise ImportError(f"{_LIB} not built (make -C oracle)")
        L = C.CDLL(str(_LIB))
        P, S, U64, F, I = C.c_void_p, C.c_size_t, C.c_uint64, C.c_float, C.c_int
        L.tr_fill_bf16.argtypes = [P, S, U64, U64, F]
        L.tr_synth_value.argtypes = [U64, U64, U64, F]
        L.tr_synth_value.restype = F
        L.tr_gemm_rows.argtypes = [P, P, P, I, I, I, P, I]
        L.tr_axpy_bf16.argtypes = [P, P, F, S, S]
        L.tr_bias_gelu.argtypes = [P, P, P, I, I]
        L.tr_silu_mul.argtypes = [P, P, I, I]
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def synth_bf16(n: int, seed: int, tensor: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint16)
    lib().tr_fill_bf16(_p(out), n, seed, tensor, scale)
    return out


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def gemm_rows(A: np.ndarray, W: np.ndarray, rows, N: int, K: int) -> np.ndarray:
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int32))
    out = np.empty((len(rows), N), dtype=np.float32)
    lib().tr_gemm_rows(_p(A), _p(W), _p(out), 0, N, K, _p(rows), len(rows))
    return out


def axpy(y: np.ndarray, x: np.ndarray, alpha: float, begin: int = 0, end: int | None = None) -> np.ndarray:
    y = y.copy()
    lib().tr_axpy_bf16(_p(y), _p(x), alpha, begin, len(y) if end is None else end)
    return y


def bias_gelu(x: np.ndarray, bias: np.ndarray, M: int, N: int) -> np.ndarray:
    out = np.empty(M * N, dtype=np.uint16)
    lib().tr_bias_gelu(_p(x), _p(bias), _p(out), M, N)
    return out


def silu_mul(x: np.ndarray, M: int, N: int) -> np.ndarray:
    """out[m, n] = silu(x[m, n]) * x[m, N + n] for x = [M x 2N] bf16 (oracle/tenant_ref.c)."""
    out = np.empty(M * N, dtype=np.uint16)
    lib().tr_silu_mul(_p(x), _p(out), M, N)
    return out
