"""ctypes bindings of the in-tree native libraries (no torch types cross the boundary).

libmicroslice.so : scheduler core / replay C-ABI      (include/ms_replay.h)
libms_b200.so    : sm_100a device layer + live runtime (include/ms_b200.h)

Both are built in-tree by ``make`` (``__graft_entry__.build()``).  Loading fails loudly
if a library is missing: there is no Python or CPU fallback for the product path.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_DIR = _PKG / "lib"

MS_OK, MS_E_ARG, MS_E_VALIDATION, MS_E_ENGINE, MS_E_CAPACITY = 0, -1, -2, -3, -4
MS_RUN_NDJSON, MS_RUN_REPORT, MS_RUN_DELAYS, MS_RUN_ROWS = 1, 2, 4, 8


class ValidationError(ValueError):
    """Mirror of microslice::ValidationError (SPEC exit code 2)."""


class EngineError(RuntimeError):
    """Mirror of microslice::EngineError (SPEC exit code 3)."""


class MsBox(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("ox", "oy", "oz", "sx", "sy", "sz")]

    def astuple(self):
        return (self.ox, self.oy, self.oz, self.sx, self.sy, self.sz)


class MsSplitPlan(C.Structure):
    _fields_ = [("blocks_per_slice", C.c_int64), ("predicted_slice_time_ns", C.c_int64),
                ("cap_ns", C.c_int64), ("memory_bound", C.c_int32), ("uncappable", C.c_int32),
                ("n_slices", C.c_int64)]


def _load(name: str) -> C.CDLL:
    path = LIB_DIR / name
    if not path.exists():
        raise ImportError(f"{path} is not built; run `make` (or __graft_entry__.build())")
    return C.CDLL(str(path), mode=C.RTLD_LOCAL)


_core = None


def core() -> C.CDLL:
    global _core
    if _core is None:
        lib = _load("libmicroslice.so")
        P, S, I64, U64, D, I32 = C.c_char_p, C.c_size_t, C.c_int64, C.c_uint64, C.c_double, C.c_int32
        sig = {
            "ms_splitmix64": (U64, [U64]),
            "ms_hash_combine": (U64, [U64, U64]),
            "ms_hash_str": (U64, [P, S]),
            "ms_u01_from_key": (D, [U64]),
            "ms_dist_sample": (C.c_int, [P, C.POINTER(D), S, C.POINTER(I64), P, S]),
            "ms_dist_sample_keyed": (C.c_int, [P, C.POINTER(U64), S, C.POINTER(I64), P, S]),
            "ms_dist_mean": (C.c_int, [P, C.POINTER(I64), P, S]),
            "ms_concurrent_capacity": (C.c_int, [P, P, C.c_int, C.POINTER(I64), P, S]),
            "ms_exec_time_model": (C.c_int, [P, P, I64, D, C.c_int, C.POINTER(I64), P, S]),
            "ms_find_optimal_split": (C.c_int, [P, P, D, I64, C.c_int, C.c_int, C.POINTER(MsSplitPlan),
                                                C.POINTER(MsBox), S, P, S]),
            "ms_slice_boxes": (C.c_int, [I32, I32, I32, I64, C.c_int, C.POINTER(MsBox), S, C.POINTER(S)]),
            "ms_consolidate": (C.c_int, [I32, I32, I32, C.POINTER(MsBox), S, C.POINTER(MsBox), S,
                                         C.POINTER(S)]),
            "ms_predict_interval": (I64, [C.POINTER(I64), S, D, I32, I64]),
            "ms_tick_interval": (I64, [I64, I64]),
            "ms_consolidation_prefix": (C.c_int, [P, P, C.POINTER(I64), S, I64, D, C.POINTER(I64), P, S]),
            "ms_percentile": (I64, [C.POINTER(I64), S, D]),
            "ms_generate_bursty_arrivals": (C.c_int, [D, D, I64, U64, I64, C.POINTER(I64), S, C.POINTER(S),
                                                      P, S]),
            "ms_replay_run": (C.c_int, [P, P, C.c_int, C.POINTER(C.c_void_p), P, S]),
            "ms_replay_run_opts": (C.c_int, [P, P, P, C.c_int, C.POINTER(C.c_void_p), P, S]),
            "ms_scenario_normalize": (C.c_int, [P, C.POINTER(C.c_void_p), P, S]),
            "ms_free": (None, [C.c_void_p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _core = lib
    return _core


def check(rc: int, err: C.Array | None = None) -> None:
    if rc == MS_OK:
        return
    msg = err.value.decode(errors="replace") if err is not None else ""
    if rc == MS_E_VALIDATION:
        raise ValidationError(msg)
    if rc == MS_E_ENGINE:
        raise EngineError(msg)
    raise RuntimeError(f"microslice native call failed rc={rc}: {msg}")


def errbuf() -> C.Array:
    return C.create_string_buffer(1024)


def take_string(lib: C.CDLL, ptr: C.c_void_p, free_name: str = "ms_free") -> str:
    s = C.cast(ptr, C.c_char_p).value.decode()
    getattr(lib, free_name)(ptr)
    return s


def _js(x) -> bytes:
    return (x if isinstance(x, str) else json.dumps(x)).encode()


def replay_run(scenario, policy: str, flags: int = 0, options: dict | None = None) -> dict:
    """Engine(ScenarioSpec, Policy, EngineOptions).run() on the replay backend; returns the artifacts digest."""
    lib, err, out = core(), errbuf(), C.c_void_p()
    opts = json.dumps(options).encode() if options else None
    check(lib.ms_replay_run_opts(_js(scenario), policy.encode(), opts, flags, C.byref(out), err, len(err)), err)
    return json.loads(take_string(lib, out))
