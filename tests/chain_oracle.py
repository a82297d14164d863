"""TEST INFRASTRUCTURE: evaluate an HP op list (the ms_hp_op dicts a chain was registered
with) with the C restatement in oracle/tenant_ref.c, op by op.

Two modes, both returning per-op (normwise, elementwise) errors against the device:
  * isolated: every op's inputs are read back from the DEVICE buffers the op consumed, so
    each op is checked on its own (differences = output rounding + accumulation order);
  * chained: inputs come from the oracle's own earlier outputs (bf16-rounded between ops
    exactly like the device), so errors compound over the whole network — reported
    normwise for the final output.
Buffers are resolved by address containment (an op may read a column slice of a wider
buffer through `lda`)."""
from __future__ import annotations

import numpy as np

GEMM, BIAS_GELU, SILU_MUL, GEMM_SWIGLU = 1, 2, 5, 6
IM2COL, BIAS_ACT, MAXPOOL, AVGPOOL, ATTN, ADD_LN = 7, 8, 9, 10, 11, 12


def rnd(y):
    u = np.ascontiguousarray(y, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def errs(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    err = np.abs(got - want)
    scale = max(float(np.max(np.abs(want))), 1e-30)
    return float(np.max(err) / scale), float(np.max(err / np.maximum(np.abs(want), 1e-2 * scale)))


class ChainOracle:
    def __init__(self, T, dev, bufs: dict[str, tuple[int, int]]):
        self.T, self.dev = T, dev
        self.regions = sorted((p, n, name) for name, (p, n) in bufs.items())
        self.mem: dict[int, np.ndarray] = {}  # oracle copy of each buffer (uint16 view), by base

    def _region(self, ptr):
        for base, n, _ in self.regions:
            if base <= ptr < base + n:
                return base, n
        raise KeyError(hex(ptr))

    def device(self, ptr, count):
        base, n = self._region(ptr)
        out = np.empty(count, np.uint16)
        self.dev.d2h(out.ctypes.data, ptr, count * 2)
        return out

    def _read(self, ptr, count, chained):
        if not chained:
            return self.device(ptr, count)
        base, n = self._region(ptr)
        if base not in self.mem:
            self.mem[base] = self.device(base, n // 2)  # weights / inputs: read once
        off = (ptr - base) // 2
        return self.mem[base][off:off + count]

    def _write(self, ptr, val):
        base, n = self._region(ptr)
        if base not in self.mem:
            self.mem[base] = np.zeros(n // 2, np.uint16)
        off = (ptr - base) // 2
        self.mem[base][off:off + len(val)] = val

    def op(self, o: dict, chained: bool) -> np.ndarray:
        """Oracle output (uint16 bf16 bits, row-major [m x n]) of one op."""
        T, k, m, n = self.T, o["kind"], o["m"], o["n"]
        rd = lambda p_, cnt: self._read(p_, cnt, chained)  # noqa: E731
        if k == GEMM:
            K, lda = o["k"], o.get("lda") or o["k"]
            a = rd(o["a"], (m - 1) * lda + K).copy()
            if lda != K:
                a = np.ascontiguousarray(np.lib.stride_tricks.as_strided(a, (m, K), (lda * 2, 2))).reshape(-1)
            w = rd(o["b"], n * K)
            y = T.gemm_rows(a, w, list(range(m)), n, K)
            flags = (o.get("geo") or {}).get("flags", 0)
            if o.get("bias") or o.get("resid") or flags:  # fused epilogue on the fp32 accumulators
                y = y.astype(np.float32)
                if o.get("bias"):
                    y = y + T.bf16_to_f32(rd(o["bias"], n))[None, :]
                if o.get("resid"):
                    y = y + T.bf16_to_f32(rd(o["resid"], m * n)).reshape(m, n)
                if flags & 1:
                    y = np.maximum(y, 0.0)
                if flags & 2:
                    y = 0.5 * y * (1.0 + np.tanh(0.7978845608028654 * (y + 0.044715 * y * y * y)))
            return rnd(y.reshape(-1))
        if k == GEMM_SWIGLU:  # silu(x Wg^T) * (x Wu^T) on the fp32 accumulators, W = [Wg; Wu]
            K, lda = o["k"], o.get("lda") or o["k"]
            a = rd(o["a"], (m - 1) * lda + K)
            gu = T.gemm_rows(np.ascontiguousarray(a), rd(o["b"], 2 * n * K), list(range(m)), 2 * n, K)
            g, u = gu[:, :n].astype(np.float64), gu[:, n:].astype(np.float64)
            return rnd((g / (1.0 + np.exp(-g)) * u).reshape(-1))
        if k == BIAS_GELU:
            return T.bias_gelu(rd(o["a"], m * n), rd(o["bias"], n), m, n)
        if k == IM2COL:
            g = o["geo"]
            return T.im2col(rd(o["a"], g["h"] * g["w"] * g["cin"]), g["h"], g["w"], g["cin"], g["kh"], g["kw"],
                            g["stride"], g["pad"], m, n)
        if k == BIAS_ACT:
            resid = rd(o["b"], m * n) if o.get("b") else None
            return T.bias_act(rd(o["a"], m * n), rd(o["bias"], n), resid, m, n, bool(o["geo"].get("flags", 0) & 1))
        if k == MAXPOOL:
            g = o["geo"]
            return T.maxpool(rd(o["a"], g["h"] * g["w"] * g["cin"]), g["h"], g["w"], g["cin"], g["kh"], g["stride"],
                             g["pad"], m)
        if k == AVGPOOL:
            g = o["geo"]
            return T.avgpool(rd(o["a"], g["h"] * g["w"] * n), g["h"] * g["w"], n, m)
        if k == ATTN:
            return T.attention(rd(o["a"], m * 3 * n), m, n)
        if k == ADD_LN:
            return T.add_ln(rd(o["a"], m * n), rd(o["b"], m * n), rd(o["bias"], 2 * n), m, n)
        raise ValueError(f"op kind {k}")

    def run(self, ops: list[dict], chained: bool, check=None):
        """Evaluate all ops; `check(i, got, want)` is called per op with the device output
        and the oracle output (both uint16).  Returns the oracle output of the last op."""
        out = None
        for i, o in enumerate(ops):
            out = self.op(o, chained)
            if chained:
                self._write(o["c"], out)
            if check is not None:
                check(i, self.device(o["c"], len(out)), out)
        return out
