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
        L.tr_im2col.argtypes = [P, P, I, I, I, I, I, I, I, I, I]
        L.tr_bias_act.argtypes = [P, P, P, P, I, I, I]
        L.tr_maxpool.argtypes = [P, P, I, I, I, I, I, I, I]
        L.tr_avgpool.argtypes = [P, P, I, I, I]
        L.tr_attention.argtypes = [P, P, I, I]
        L.tr_add_ln.argtypes = [P, P, P, P, I, I]
        L.tr_optim.argtypes = [P, P, P, P, S, S, I, F, F, F, F, F, F, F]
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


# ---- config-2 / config-3 glue ops (oracle/tenant_ref.c; device: hp_ops.cuh) -------------
def im2col(x: np.ndarray, h: int, w: int, cin: int, kh: int, kw: int, stride: int, pad: int,
           m_pad: int, n_pad: int) -> np.ndarray:
    out = np.empty(m_pad * n_pad, dtype=np.uint16)
    lib().tr_im2col(_p(np.ascontiguousarray(x)), _p(out), h, w, cin, kh, kw, stride, pad, m_pad, n_pad)
    return out


def bias_act(x: np.ndarray, bias: np.ndarray, resid, m: int, n: int, relu: bool) -> np.ndarray:
    out = np.empty(m * n, dtype=np.uint16)
    r = None if resid is None else np.ascontiguousarray(resid)
    lib().tr_bias_act(_p(np.ascontiguousarray(x)), _p(bias), None if r is None else _p(r), _p(out), m, n, int(relu))
    return out


def maxpool(x: np.ndarray, h: int, w: int, c: int, k: int, stride: int, pad: int, m_pad: int) -> np.ndarray:
    out = np.empty(m_pad * c, dtype=np.uint16)
    lib().tr_maxpool(_p(np.ascontiguousarray(x)), _p(out), h, w, c, k, stride, pad, m_pad)
    return out


def avgpool(x: np.ndarray, rows: int, n: int, m_pad: int) -> np.ndarray:
    out = np.empty(m_pad * n, dtype=np.uint16)
    lib().tr_avgpool(_p(np.ascontiguousarray(x)), _p(out), rows, n, m_pad)
    return out


def attention(qkv: np.ndarray, s: int, d: int) -> np.ndarray:
    out = np.empty(s * d, dtype=np.uint16)
    lib().tr_attention(_p(np.ascontiguousarray(qkv)), _p(out), s, d)
    return out


def add_ln(x: np.ndarray, resid: np.ndarray, gb: np.ndarray, m: int, n: int) -> np.ndarray:
    out = np.empty(m * n, dtype=np.uint16)
    lib().tr_add_ln(_p(np.ascontiguousarray(x)), _p(np.ascontiguousarray(resid)), _p(gb), _p(out), m, n)
    return out


def synth_f32(n: int, seed: int, tensor: int, scale: float = 1.0) -> np.ndarray:
    """fp32 tensor of the bf16 synthetic values (device: ms_fill_synth_f32)."""
    return bf16_to_f32(synth_bf16(n, seed, tensor, scale)).copy()


def optim(p, m, v, g, mode, lr, b1, b2, eps, wd, c1, c2, begin=0, end=None):
    """In-place optimizer step over fp32 p / m / v (v ignored by SGD) and bf16 g."""
    end = len(p) if end is None else end
    lib().tr_optim(_p(p), _p(m), _p(v), _p(g), begin, end, mode, lr, b1, b2, eps, wd, c1, c2)
