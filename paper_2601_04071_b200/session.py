"""Python binding of the external-tenant live session (include/ms_session.h).

An HP tenant (e.g. a decode loop) submits its pre-registered chains and announces its
CPU-side bubbles; the session's scheduler thread harvests them with preemptible LP kernels.

    with LiveSession(dev, [lp.id], chain) as s:
        for token in range(n):
            seq = s.submit(chain)
            s.wait(seq)
            s.hint(300_000)          # sampling + detokenize, ~300 us
            ...CPU work...
    report = s.report
"""
from __future__ import annotations

import ctypes as C
import json

from .device import Device, HpTimes, _ck, lib as dev_lib


def _lib():
    L = dev_lib()
    if not hasattr(L, "_ms_session_sig"):
        P, I, U32, I64 = C.c_void_p, C.c_int, C.c_uint32, C.c_int64
        L.ms_session_start.restype = I
        L.ms_session_start.argtypes = [P, C.POINTER(I), I, I, C.c_char_p, C.POINTER(P)]
        L.ms_session_hp_prepare.argtypes = [P, I]
        L.ms_session_hp_submit.argtypes = [P, I, C.POINTER(U32)]
        L.ms_session_hp_wait.argtypes = [P, U32, I64, C.POINTER(HpTimes)]
        L.ms_session_hint.argtypes = [P, I64]
        L.ms_session_stop.argtypes = [P, C.POINTER(P)]
        L.ms_live_free.argtypes = [P]
        L._ms_session_sig = True
    return L


class LiveSession:
    def __init__(self, dev: Device, lp_ids: list[int], hp_chain: int, options: dict | None = None):
        self.dev, self._h, self.report = dev, C.c_void_p(), None
        L = _lib()
        ids = (C.c_int * len(lp_ids))(*lp_ids)
        _ck(L.ms_session_start(dev._h, ids, len(lp_ids), hp_chain, json.dumps(options or {}).encode(),
                               C.byref(self._h)))

    def prepare(self, chain: int):
        _ck(_lib().ms_session_hp_prepare(self._h, chain))

    def submit(self, chain: int) -> int:
        seq = C.c_uint32()
        _ck(_lib().ms_session_hp_submit(self._h, chain, C.byref(seq)))
        return seq.value

    def wait(self, seq: int, timeout_s: float = 10.0) -> dict:
        t = HpTimes()
        _ck(_lib().ms_session_hp_wait(self._h, seq, int(timeout_s * 1e9), C.byref(t)))
        return t.asdict()

    def hint(self, predicted_ns: int):
        _ck(_lib().ms_session_hint(self._h, int(predicted_ns)))

    def stop(self) -> dict:
        if self._h:
            out = C.c_void_p()
            L = _lib()
            _ck(L.ms_session_stop(self._h, C.byref(out)))
            self.report = json.loads(C.cast(out, C.c_char_p).value.decode())
            L.ms_live_free(out)
            self._h = C.c_void_p()
        return self.report

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.stop()
