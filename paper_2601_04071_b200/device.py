"""ctypes view of libms_b200.so (include/ms_b200.h): the sm_100a device layer.

Plain C types cross the boundary (device pointers are ints).  Any failure raises
DeviceError carrying ms_last_error(); there is no CPU fallback — a missing library or
GPU is an error, never a silent downgrade.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native

MS_LP_GEMM, MS_LP_AXPY, MS_LP_OPTIM = 1, 2, 3
MS_HP_GEMM, MS_HP_BIAS_GELU, MS_HP_H2D, MS_HP_D2H = 1, 2, 3, 4
MS_HP_SILU_MUL, MS_HP_GEMM_SWIGLU = 5, 6
MS_HP_IM2COL, MS_HP_BIAS_ACT, MS_HP_MAXPOOL, MS_HP_AVGPOOL, MS_HP_ATTN, MS_HP_ADD_LN = 7, 8, 9, 10, 11, 12


class DeviceError(RuntimeError):
    pass


class DevInfo(C.Structure):
    _fields_ = [("ordinal", C.c_int32), ("sm_count", C.c_int32), ("cc_major", C.c_int32),
                ("cc_minor", C.c_int32), ("stream_memops", C.c_int32), ("prio_low", C.c_int32),
                ("prio_high", C.c_int32), ("hbm_bytes", C.c_int64), ("name", C.c_char * 64)]


class LpDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("block_n", C.c_int32), ("group_m", C.c_int32),
                ("tile_elems", C.c_int32), ("ctas_per_sm", C.c_int32), ("split_k", C.c_int32),
                ("a", C.c_uint64), ("b", C.c_uint64), ("c", C.c_uint64),
                ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64),
                ("x", C.c_uint64), ("y", C.c_uint64), ("alpha", C.c_float), ("pad2", C.c_float),
                ("n_elems", C.c_int64), ("opt_mode", C.c_int32), ("opt", C.c_float * 7)]


class LpStatus(C.Structure):
    _fields_ = [("run_id", C.c_uint64), ("begin", C.c_uint64), ("end", C.c_uint64),
                ("redo_in", C.c_uint64), ("cursor", C.c_uint64), ("redo_count", C.c_uint64),
                ("tiles_done", C.c_uint64), ("preempted", C.c_int32), ("done", C.c_int32),
                ("t_launch_host", C.c_int64), ("t_start", C.c_uint64), ("t_seen", C.c_uint64),
                ("t_exit", C.c_uint64), ("t_free", C.c_uint64)]

    def asdict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class HpGeo(C.Structure):
    _fields_ = [("h", C.c_int32), ("w", C.c_int32), ("cin", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32),
                ("stride", C.c_int32), ("pad", C.c_int32), ("flags", C.c_int32)]


class HpOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("block_n", C.c_int32), ("a", C.c_uint64), ("b", C.c_uint64),
                ("c", C.c_uint64), ("bias", C.c_uint64), ("m", C.c_int64), ("n", C.c_int64),
                ("k", C.c_int64), ("split_k", C.c_int32), ("b_layout", C.c_int32), ("lda", C.c_int64),
                ("geo", HpGeo), ("resid", C.c_uint64)]

    @classmethod
    def from_dict(cls, o: dict) -> "HpOp":
        o = dict(o)
        geo = o.pop("geo", None)
        op = cls(**o)
        if geo:
            op.geo = HpGeo(**geo)
        return op


class MsEvent(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("t_ns", C.c_uint64), ("kind", C.c_uint32), ("id", C.c_uint32),
                ("a", C.c_uint64), ("b", C.c_uint64)]


EVENT_KINDS = {1: "lp_start", 2: "lp_seen", 3: "lp_exit", 4: "hp_first", 5: "hp_done", 6: "gate"}


class HpTimes(C.Structure):
    _fields_ = [("seq", C.c_uint32), ("done", C.c_uint32), ("t_gate", C.c_uint64),
                ("t_first_cta", C.c_uint64), ("t_done", C.c_uint64)]

    def asdict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _native.core()  # libms_b200 links libmicroslice; make sure it is resolvable first
        L = _native._load("libms_b200.so")
        P, I, U32, U64, I64, F = C.c_void_p, C.c_int, C.c_uint32, C.c_uint64, C.c_int64, C.c_float
        sig = {
            "ms_dev_open": (I, [I, C.POINTER(P)]), "ms_dev_close": (I, [P]),
            "ms_dev_get_info": (I, [P, C.POINTER(DevInfo)]), "ms_dev_sync": (I, [P]),
            "ms_last_error": (C.c_char_p, []), "ms_host_now_ns": (I64, []),
            "ms_mem_alloc": (I, [P, C.c_size_t, C.POINTER(U64)]), "ms_mem_free": (I, [P, U64]),
            "ms_host_alloc": (I, [P, C.c_size_t, C.POINTER(U64)]), "ms_host_free": (I, [P, U64]),
            "ms_memcpy_h2d": (I, [P, U64, P, C.c_size_t]), "ms_memcpy_d2h": (I, [P, P, U64, C.c_size_t]),
            "ms_memset": (I, [P, U64, I, C.c_size_t]),
            "ms_fill_synth_bf16": (I, [P, U64, U64, U64, U64, F]),
            "ms_fill_synth_f32": (I, [P, U64, U64, U64, U64, F]),
            "ms_lp_register": (I, [P, C.POINTER(LpDesc), C.POINTER(I), C.POINTER(U64)]),
            "ms_lp_run": (I, [P, I, U64, U64, U64]), "ms_lp_set_budget": (I, [P, I, U64]),
            "ms_lp_set_slow_tiles": (I, [P, I, C.c_char_p, U64, I, I]),
            "ms_lp_poll": (I, [P, I, C.POINTER(LpStatus)]),
            "ms_lp_wait": (I, [P, I, I64, C.POINTER(LpStatus)]), "ms_lp_reset": (I, [P, I]),
            "ms_preempt_raise": (I, [P, C.POINTER(U32), C.POINTER(I64)]), "ms_preempt_epoch": (U32, [P]),
            "ms_hp_register_chain": (I, [P, C.POINTER(HpOp), I, C.POINTER(I)]),
            "ms_hp_arm": (I, [P, I, U32]), "ms_hp_ring": (I, [P, U32, C.POINTER(I64)]),
            "ms_hp_next_seq": (U32, [P]), "ms_lp_total_tiles": (U64, [P, I]), "ms_lp_tile_ctas": (I, [P, I]), "ms_lp_progress": (U64, [P, I]),
            "ms_lp_run_ex": (I, [P, I, U64, U64, U64, I]), "ms_lp_unregister": (I, [P, I]),
            "ms_debug_stamps": (I, [P, I, C.POINTER(C.c_ulonglong), C.c_size_t]),
            "ms_set_lp_sm_reserve": (I, [P, I]),
            "ms_hp_set_fused": (I, [P, I]),
            "ms_hp_unregister_chain": (I, [P, I]),
            "ms_hp_chain_info": (I, [P, I, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "ms_hp_launch_direct": (I, [P, I, U32]),
            "ms_hp_poll": (I, [P, I, U32, C.POINTER(HpTimes)]),
            "ms_hp_wait": (I, [P, I, U32, I64, C.POINTER(HpTimes)]),
            "ms_clock_calibrate": (I, [P, I, C.POINTER(I64), C.POINTER(I64)]),
            "ms_lp_time_full": (I, [P, I, I, C.POINTER(F)]),
            "ms_lp_time_range": (I, [P, I, U64, U64, I, C.POINTER(F)]),
            "ms_hp_time_chain": (I, [P, I, I, C.POINTER(F)]),
            "ms_trace_enable": (I, [P, C.c_size_t]),
            "ms_trace_drain": (I, [P, C.POINTER(MsEvent), C.c_size_t, C.POINTER(U64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def _ck(rc: int) -> int:
    if rc < 0:
        raise DeviceError(f"ms_b200 rc={rc}: {lib().ms_last_error().decode(errors='replace')}")
    return rc


def host_now_ns() -> int:
    return lib().ms_host_now_ns()


@dataclass
class LpKernel:
    id: int
    total_tiles: int
    tile_ctas: int = 1  # SMs one tile occupies (2: GEMM on CTA pairs)


class Device:
    """One B200 under this process's scheduler (one ms_dev per GPU, no sharing)."""

    def __init__(self, ordinal: int = 0):
        self._h = C.c_void_p()
        _ck(lib().ms_dev_open(ordinal, C.byref(self._h)))
        info = DevInfo()
        _ck(lib().ms_dev_get_info(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in DevInfo._fields_}
        self.info["name"] = info.name.decode()

    def close(self):
        if self._h:
            lib().ms_dev_close(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- memory
    def alloc(self, nbytes: int) -> int:
        p = C.c_uint64()
        _ck(lib().ms_mem_alloc(self._h, nbytes, C.byref(p)))
        return p.value

    def host_alloc(self, nbytes: int) -> int:
        p = C.c_uint64()
        _ck(lib().ms_host_alloc(self._h, nbytes, C.byref(p)))
        return p.value

    def host_free(self, ptr: int):
        _ck(lib().ms_host_free(self._h, ptr))

    def free(self, ptr: int):
        _ck(lib().ms_mem_free(self._h, ptr))

    def h2d(self, dst: int, src_ptr: int, nbytes: int):
        _ck(lib().ms_memcpy_h2d(self._h, dst, src_ptr, nbytes))

    def d2h(self, dst_ptr: int, src: int, nbytes: int):
        _ck(lib().ms_memcpy_d2h(self._h, dst_ptr, src, nbytes))

    def memset(self, dst: int, value: int, nbytes: int):
        _ck(lib().ms_memset(self._h, dst, value, nbytes))

    def fill_synth(self, dst: int, n: int, seed: int, tensor: int, scale: float = 1.0):
        _ck(lib().ms_fill_synth_bf16(self._h, dst, n, seed, tensor, scale))

    def fill_synth_f32(self, dst: int, n: int, seed: int, tensor: int, scale: float = 1.0):
        _ck(lib().ms_fill_synth_f32(self._h, dst, n, seed, tensor, scale))

    def sync(self):
        _ck(lib().ms_dev_sync(self._h))

    # ---- LP
    def lp_register_gemm(self, a: int, b: int, c: int, m: int, n: int, k: int, block_n: int = 256,
                         group_m: int = 16, split_k: int = 1) -> LpKernel:
        """split_k > 1: work unit = (tile, k-slice), the tile's last unit reduces the fp32
        partials in slice order (total_tiles counts units)."""
        d = LpDesc(kind=MS_LP_GEMM, block_n=block_n, group_m=group_m, a=a, b=b, c=c, m=m, n=n, k=k,
                   split_k=split_k)
        return self._lp_register(d)

    def lp_register_axpy(self, x: int, y: int, n_elems: int, alpha: float, tile_elems: int = 8192,
                         ctas_per_sm: int = 1) -> LpKernel:
        d = LpDesc(kind=MS_LP_AXPY, tile_elems=tile_elems, ctas_per_sm=ctas_per_sm, x=x, y=y,
                   alpha=alpha, n_elems=n_elems)
        return self._lp_register(d)

    def lp_register_optim(self, params: int, m1: int, m2: int, grads: int, n_elems: int, mode: int = 0,
                          lr: float = 1e-4, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                          wd: float = 0.01, c1: float = 1.0, c2: float = 1.0, tile_elems: int = 4096) -> LpKernel:
        """Optimizer step streamer (MS_LP_OPTIM): mode 0 AdamW over fp32 params / moments and
        bf16 grads, mode 1 SGD momentum (beta1 = momentum, m2 unused)."""
        d = LpDesc(kind=MS_LP_OPTIM, tile_elems=tile_elems, a=params, b=m1, c=m2, x=grads, n_elems=n_elems,
                   opt_mode=mode)
        for i, v in enumerate((lr, beta1, beta2, eps, wd, c1, c2)):
            d.opt[i] = v
        return self._lp_register(d)

    def _lp_register(self, d: LpDesc) -> LpKernel:
        kid, tiles = C.c_int(), C.c_uint64()
        _ck(lib().ms_lp_register(self._h, C.byref(d), C.byref(kid), C.byref(tiles)))
        return LpKernel(kid.value, tiles.value, _ck(lib().ms_lp_tile_ctas(self._h, kid.value)))

    def lp_set_slow_tiles(self, k: LpKernel, slow_groups, tiles_per_group: int, max_inflight: int = 8):
        """Memory tier: bound the streamer's in-flight tiles over off-device chunks
        (include/ms_b200.h ms_lp_set_slow_tiles).  slow_groups=None disables."""
        if slow_groups is None:
            _ck(lib().ms_lp_set_slow_tiles(self._h, k.id, None, 0, 0, 0))
            return
        b = bytes(1 if g else 0 for g in slow_groups)
        _ck(lib().ms_lp_set_slow_tiles(self._h, k.id, b, len(b), tiles_per_group, max_inflight))

    def lp_unregister(self, k: LpKernel):
        _ck(lib().ms_lp_unregister(self._h, k.id))

    def lp_run(self, k: LpKernel, begin: int, end: int, budget: int | None = None):
        _ck(lib().ms_lp_run(self._h, k.id, begin, end, end if budget is None else budget))

    def lp_set_budget(self, k: LpKernel, budget: int):
        _ck(lib().ms_lp_set_budget(self._h, k.id, budget))

    def lp_poll(self, k: LpKernel) -> dict | None:
        st = LpStatus()
        return st.asdict() if _ck(lib().ms_lp_poll(self._h, k.id, C.byref(st))) else None

    def lp_wait(self, k: LpKernel, timeout_s: float = 30.0) -> dict:
        st = LpStatus()
        _ck(lib().ms_lp_wait(self._h, k.id, int(timeout_s * 1e9), C.byref(st)))
        return st.asdict()

    def lp_reset(self, k: LpKernel):
        _ck(lib().ms_lp_reset(self._h, k.id))

    # ---- device-side event trace (include/ms_b200.h ms_trace_*)
    def trace_enable(self, capacity: int = 1 << 14):
        _ck(lib().ms_trace_enable(self._h, capacity))

    def trace_drain(self, max_events: int = 1 << 14) -> tuple[list[dict], int]:
        """Events written by the kernels since the last drain (oldest first) and the running
        count of events overwritten before they were drained."""
        buf = (MsEvent * max_events)()
        lost = C.c_uint64()
        n = _ck(lib().ms_trace_drain(self._h, buf, max_events, C.byref(lost)))
        evs = [{"seq": e.seq, "t_ns": e.t_ns, "kind": EVENT_KINDS.get(e.kind, e.kind), "id": e.id, "a": e.a, "b": e.b}
               for e in buf[:n]]
        return evs, lost.value

    def lp_time_full(self, k: LpKernel, reps: int = 5) -> float:
        ms = C.c_float()
        _ck(lib().ms_lp_time_full(self._h, k.id, reps, C.byref(ms)))
        return ms.value

    def lp_time_range(self, k: LpKernel, begin: int, end: int, reps: int = 3) -> float:
        """CUDA-event time (ms) of an LP run over tiles [begin, end)."""
        ms = C.c_float()
        _ck(lib().ms_lp_time_range(self._h, k.id, begin, end, reps, C.byref(ms)))
        return ms.value

    def set_lp_sm_reserve(self, n: int):
        _ck(lib().ms_set_lp_sm_reserve(self._h, n))

    def hp_set_fused(self, mode):
        """1/True: fused launch per chain (cluster split-K when it fits, default);
        2: fused, global split-K reduction; 0/False: one kernel per HP op."""
        _ck(lib().ms_hp_set_fused(self._h, int(mode)))

    def hp_chain_info(self, chain: int) -> dict:
        g, c = C.c_int(), C.c_int()
        _ck(lib().ms_hp_chain_info(self._h, chain, C.byref(g), C.byref(c)))
        return {"fused_grid": g.value, "cluster": c.value}

    def debug_stamps(self, enable: bool, n_cta: int = 148):
        if enable:
            _ck(lib().ms_debug_stamps(self._h, 1, None, 0))
            return None
        buf = (C.c_ulonglong * (n_cta * 8))()
        _ck(lib().ms_debug_stamps(self._h, 0, buf, n_cta * 8))
        return [list(buf[i * 8:(i + 1) * 8]) for i in range(n_cta)]

    def debug_stamps_ext(self, n_cta: int = 148) -> list[list[int]]:
        """Read (and disarm) the extended [cta][64] stamp block (fused HP chain kernel)."""
        buf = (C.c_ulonglong * (2048 + n_cta * 64))()
        _ck(lib().ms_debug_stamps(self._h, 0, buf, 2048 + n_cta * 64))
        return [list(buf[2048 + i * 64:2048 + (i + 1) * 64]) for i in range(n_cta)]

    # ---- preemption
    def preempt_raise(self) -> tuple[int, int]:
        e, t = C.c_uint32(), C.c_int64()
        _ck(lib().ms_preempt_raise(self._h, C.byref(e), C.byref(t)))
        return e.value, t.value

    def epoch(self) -> int:
        return lib().ms_preempt_epoch(self._h)

    # ---- HP
    def hp_register_chain(self, ops: list[dict]) -> int:
        arr = (HpOp * len(ops))(*[HpOp.from_dict(o) for o in ops])
        cid = C.c_int()
        _ck(lib().ms_hp_register_chain(self._h, arr, len(ops), C.byref(cid)))
        return cid.value

    def hp_unregister_chain(self, chain: int):
        _ck(lib().ms_hp_unregister_chain(self._h, chain))

    def hp_next_seq(self) -> int:
        return lib().ms_hp_next_seq(self._h)

    def hp_arm(self, chain: int, seq: int):
        _ck(lib().ms_hp_arm(self._h, chain, seq))

    def hp_ring(self, seq: int) -> int:
        t = C.c_int64()
        _ck(lib().ms_hp_ring(self._h, seq, C.byref(t)))
        return t.value

    def hp_launch_direct(self, chain: int, seq: int):
        _ck(lib().ms_hp_launch_direct(self._h, chain, seq))

    def hp_poll(self, chain: int, seq: int) -> dict | None:
        t = HpTimes()
        return t.asdict() if _ck(lib().ms_hp_poll(self._h, chain, seq, C.byref(t))) else None

    def hp_wait(self, chain: int, seq: int, timeout_s: float = 10.0) -> dict:
        t = HpTimes()
        _ck(lib().ms_hp_wait(self._h, chain, seq, int(timeout_s * 1e9), C.byref(t)))
        return t.asdict()

    def hp_time_chain(self, chain: int, reps: int = 20) -> float:
        ms = C.c_float()
        _ck(lib().ms_hp_time_chain(self._h, chain, reps, C.byref(ms)))
        return ms.value

    # ---- clocks
    def calibrate(self, rounds: int = 300) -> tuple[int, int]:
        off, rtt = C.c_int64(), C.c_int64()
        _ck(lib().ms_clock_calibrate(self._h, rounds, C.byref(off), C.byref(rtt)))
        return off.value, rtt.value
