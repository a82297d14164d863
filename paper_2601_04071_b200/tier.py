"""Python binding of the live memory tier (include/ms_tier.h).

    tier = MemoryTier(dev, {"hbm_gb": 0.3})                  # budget in local HBM
    x = tier.alloc(task=1, nbytes=256 << 20)                  # LP buffer: spills when full
    h = tier.alloc(task=0, nbytes=64 << 20, high_priority=True)  # pinned; displaces LP chunks
    tier.chunks(x)   # [("local"|"peer"|"dram", peer, owner, pinned), ...]

Buffers are ordinary device pointers (one VMM range each) for ms_lp_register & co.
"""
from __future__ import annotations

import ctypes as C
import json

from .device import Device, _ck, lib as dev_lib

TIERS = ("local", "peer", "dram")


class TierChunk(C.Structure):
    _fields_ = [("tier", C.c_int32), ("peer", C.c_int32), ("owner", C.c_int32), ("pinned", C.c_int32)]


class TierStats(C.Structure):
    _fields_ = [("local_capacity_chunks", C.c_int64), ("local_used_chunks", C.c_int64),
                ("chunks_local", C.c_int64), ("chunks_peer", C.c_int64), ("chunks_dram", C.c_int64),
                ("relocations", C.c_int64), ("relocated_bytes", C.c_int64), ("relocate_copy_ns", C.c_int64),
                ("relocate_remap_ns", C.c_int64), ("probes", C.c_int64),
                ("n_links", C.c_int32), ("pad", C.c_int32)]


def _lib():
    L = dev_lib()
    if not hasattr(L, "_ms_tier_sig"):
        P, I, U64, I64 = C.c_void_p, C.c_int, C.c_uint64, C.c_int64
        L.ms_tier_open.argtypes = [P, C.c_char_p, C.POINTER(P)]
        L.ms_tier_alloc.argtypes = [P, I, I, U64, C.POINTER(U64), C.POINTER(U64)]
        L.ms_tier_chunks.argtypes = [P, U64, C.POINTER(TierChunk), U64]
        L.ms_tier_probe.argtypes = [P, I, C.POINTER(C.c_double), C.POINTER(I64)]
        L.ms_tier_get_stats.argtypes = [P, C.POINTER(TierStats)]
        L.ms_tier_free.argtypes = [P, U64]
        L.ms_tier_close.argtypes = [P]
        for f in ("ms_tier_open", "ms_tier_alloc", "ms_tier_chunks", "ms_tier_probe", "ms_tier_get_stats",
                  "ms_tier_free", "ms_tier_close"):
            getattr(L, f).restype = I
        L._ms_tier_sig = True
    return L


class MemoryTier:
    CHUNK = 2 << 20

    def __init__(self, dev: Device, options: dict | None = None):
        self.dev, self._h, self._n = dev, C.c_void_p(), {}
        _ck(_lib().ms_tier_open(dev._h, json.dumps(options or {}).encode(), C.byref(self._h)))

    def alloc(self, task: int, nbytes: int, high_priority: bool = False) -> int:
        p, n = C.c_uint64(), C.c_uint64()
        _ck(_lib().ms_tier_alloc(self._h, task, int(high_priority), nbytes, C.byref(p), C.byref(n)))
        self._n[p.value] = n.value
        return p.value

    def chunks(self, ptr: int) -> list[tuple]:
        n = self._n[ptr]
        arr = (TierChunk * n)()
        _ck(_lib().ms_tier_chunks(self._h, ptr, arr, n))
        return [(TIERS[c.tier], c.peer, c.owner, bool(c.pinned)) for c in arr]

    def off_device(self, *ptrs: int) -> list[bool]:
        """Per 2 MB chunk index: True when that chunk of ANY of the equally sized buffers
        lives off the device (the streamer's slow-tile map, ms_lp_set_slow_tiles)."""
        maps = [[c[0] != "local" for c in self.chunks(p)] for p in ptrs]
        return [any(col) for col in zip(*maps)]

    def gemm_slow_units(self, a: int, b: int, m: int, n: int, k: int, block_n: int = 256, split: int = 1,
                        group_m: int = 16, block_m: int = 128) -> list[bool]:
        """Per linear work unit of an LP GEMM (C = A B^T, A [m, k], B [n, k] bf16, K-contiguous;
        unit = tile * split + k-slice, tiles in the kernel's group-M raster, tc_gemm.cuh
        tile_coords): True when the unit's A rows or B rows (its k-slice of them) touch a chunk
        that lives off the device — the GEMM's ms_lp_set_slow_tiles map.  Single-CTA kernel:
        block_m 128, group_m 16; CTA pairs (tc_gemm2.cuh): block_m 256, block_n 256 or 512,
        group_m 8."""
        off_a = [c[0] != "local" for c in self.chunks(a)]
        off_b = [c[0] != "local" for c in self.chunks(b)]
        tm, tn, kb = m // block_m, n // block_n, k // 64
        kps = kb // split

        def touches(off, row0, rows, kb0):
            lo = (row0 * k + kb0 * 64) * 2
            hi = ((row0 + rows - 1) * k + (kb0 + kps) * 64) * 2  # (rows are contiguous runs of k)
            return any(off[lo // self.CHUNK:hi // self.CHUNK + 1])

        out = []
        for t in range(tm * tn):
            span = group_m * tn
            g = t // span
            first = g * group_m
            gm = min(tm - first, group_m)
            mb, nb = first + (t - g * span) % gm, (t - g * span) // gm
            for sl in range(split):
                out.append(touches(off_a, mb * block_m, block_m, sl * kps) or
                           touches(off_b, nb * block_n, block_n, sl * kps))
        return out

    def probe(self, link: int) -> tuple[float, int]:
        s, t = C.c_double(), C.c_int64()
        _ck(_lib().ms_tier_probe(self._h, link, C.byref(s), C.byref(t)))
        return s.value, t.value

    def stats(self) -> dict:
        st = TierStats()
        _ck(_lib().ms_tier_get_stats(self._h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in TierStats._fields_ if f != "pad"}

    def free(self, ptr: int):
        _ck(_lib().ms_tier_free(self._h, ptr))
        self._n.pop(ptr, None)

    def close(self):
        if self._h:
            _lib().ms_tier_close(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
