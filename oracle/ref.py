"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes view of the compiled REFERENCE scheduler.

oracle/_ref/libmsref.so is built by oracle/Makefile from the unmodified reference
headers (/root/reference/proj/include) plus oracle/ref_driver.cpp.  Function names and
return shapes mirror paper_2601_04071_b200.microslice so tests compare like for like.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path
from typing import Sequence

_HERE = Path(__file__).resolve().parent
REF_LIB = _HERE / "_ref" / "libmsref.so"
_U64 = (1 << 64) - 1
_lib = None


def available() -> bool:
    return REF_LIB.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not REF_LIB.exists():
            raise ImportError(f"{REF_LIB} not built (make -C oracle with /root/reference present)")
        L = C.CDLL(str(REF_LIB))
        P, S, I64, U64, D, I32 = C.c_char_p, C.c_size_t, C.c_int64, C.c_uint64, C.c_double, C.c_int32
        sig = {
            "msref_splitmix64": (U64, [U64]), "msref_hash_combine": (U64, [U64, U64]),
            "msref_hash_str": (U64, [P, S]), "msref_u01_from_key": (D, [U64]),
            "msref_dist_sample": (C.c_int, [P, C.POINTER(D), S, C.POINTER(I64), P, S]),
            "msref_dist_sample_keyed": (C.c_int, [P, C.POINTER(U64), S, C.POINTER(I64), P, S]),
            "msref_dist_mean": (C.c_int, [P, C.POINTER(I64), P, S]),
            "msref_concurrent_capacity": (C.c_int, [P, P, C.c_int, C.POINTER(I64), P, S]),
            "msref_exec_time_model": (C.c_int, [P, P, I64, D, C.c_int, C.POINTER(I64), P, S]),
            "msref_find_optimal_split": (C.c_int, [P, P, D, I64, C.c_int, C.c_int, C.POINTER(I64),
                                                   C.POINTER(I32), S, P, S]),
            "msref_slice_boxes": (C.c_int, [I32, I32, I32, I64, C.c_int, C.POINTER(I32), S, C.POINTER(S)]),
            "msref_consolidate": (C.c_int, [I32, I32, I32, C.POINTER(I32), S, C.POINTER(I32), S, C.POINTER(S)]),
            "msref_predict_interval": (I64, [C.POINTER(I64), S, D, I32, I64]),
            "msref_tick_interval": (I64, [I64, I64]),
            "msref_consolidation_prefix": (C.c_int, [P, P, C.POINTER(I64), S, I64, D, C.POINTER(I64), P, S]),
            "msref_percentile": (I64, [C.POINTER(I64), S, D]),
            "msref_generate_bursty_arrivals": (C.c_int, [D, D, I64, U64, I64, C.POINTER(I64), S, C.POINTER(S),
                                                         P, S]),
            "msref_replay_run": (C.c_int, [P, P, C.c_int, C.POINTER(C.c_void_p), P, S]),
            "msref_replay_run_opts": (C.c_int, [P, P, P, C.c_int, C.POINTER(C.c_void_p), P, S]),
            "msref_parallel_runs": (C.c_int, [P, P, C.c_int, C.POINTER(D), P, S]),
            "msref_free": (None, [C.c_void_p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, rc: int, msg: str):
        super().__init__(f"rc={rc}: {msg}")
        self.rc = rc


def _chk(rc, err):
    if rc != 0:
        raise RefError(rc, err.value.decode(errors="replace"))


def _j(x) -> bytes:
    return (x if isinstance(x, str) else json.dumps(x)).encode()


def splitmix64(x): return lib().msref_splitmix64(x & _U64)
def hash_combine(a, b): return lib().msref_hash_combine(a & _U64, b & _U64)
def hash_str(s: str):
    b = s.encode()
    return lib().msref_hash_str(b, len(b))
def u01_from_key(k): return lib().msref_u01_from_key(k & _U64)


def dist_sample(dist, us):
    n = len(us)
    out, err = (C.c_int64 * n)(), C.create_string_buffer(1024)
    _chk(lib().msref_dist_sample(_j(dist), (C.c_double * n)(*us), n, out, err, 1024), err)
    return list(out)


def dist_sample_keyed(dist, keys):
    n = len(keys)
    out, err = (C.c_int64 * n)(), C.create_string_buffer(1024)
    _chk(lib().msref_dist_sample_keyed(_j(dist), (C.c_uint64 * n)(*[k & _U64 for k in keys]), n, out, err,
                                       1024), err)
    return list(out)


def dist_mean(dist):
    out, err = C.c_int64(), C.create_string_buffer(1024)
    _chk(lib().msref_dist_mean(_j(dist), C.byref(out), err, 1024), err)
    return out.value


def concurrent_capacity(gpu, kernel, rounding=0):
    out, err = C.c_int64(), C.create_string_buffer(1024)
    _chk(lib().msref_concurrent_capacity(_j(gpu), _j(kernel), rounding, C.byref(out), err, 1024), err)
    return out.value


def exec_time_model(gpu, kernel, n_blocks, load=0.0, rounding=0):
    out, err = C.c_int64(), C.create_string_buffer(1024)
    _chk(lib().msref_exec_time_model(_j(gpu), _j(kernel), n_blocks, load, rounding, C.byref(out), err, 1024),
         err)
    return out.value


def find_optimal_split(gpu, kernel, epsilon=0.02, cap_ns=400_000, square_tiling=False, rounding=0):
    plan, err = (C.c_int64 * 6)(), C.create_string_buffer(1024)
    L = lib()
    _chk(L.msref_find_optimal_split(_j(gpu), _j(kernel), epsilon, cap_ns, int(square_tiling), rounding, plan,
                                    None, 0, err, 1024), err)
    n = plan[5]
    boxes = (C.c_int32 * (6 * max(1, n)))()
    _chk(L.msref_find_optimal_split(_j(gpu), _j(kernel), epsilon, cap_ns, int(square_tiling), rounding, plan,
                                    boxes, n, err, 1024), err)
    return {"blocks_per_slice": plan[0], "predicted_slice_time": plan[1], "cap": plan[2],
            "memory_bound": bool(plan[3]), "uncappable": bool(plan[4]),
            "slices": [tuple(boxes[6 * i: 6 * i + 6]) for i in range(n)]}


def _boxes(fn, *args):
    n = C.c_size_t()
    rc = fn(*args, None, 0, C.byref(n))
    if rc not in (0, -4):
        raise RefError(rc, "")
    out = (C.c_int32 * (6 * max(1, n.value)))()
    rc = fn(*args, out, n.value, C.byref(n))
    if rc != 0:
        raise RefError(rc, "")
    return [tuple(out[6 * i: 6 * i + 6]) for i in range(n.value)]


def slice_boxes(grid, bps, square_tiling=False):
    return _boxes(lib().msref_slice_boxes, grid[0], grid[1], grid[2], bps, int(square_tiling))


def consolidate(grid, pending):
    flat = [v for b in pending for v in b]
    arr = (C.c_int32 * max(1, len(flat)))(*flat)
    return _boxes(lib().msref_consolidate, grid[0], grid[1], grid[2], arr, len(pending))


def predict_interval(gaps, alpha=0.3, k=8, fallback=2_000_000):
    return lib().msref_predict_interval((C.c_int64 * max(1, len(gaps)))(*gaps), len(gaps), alpha, k, fallback)


def tick_interval(p, l): return lib().msref_tick_interval(p, l)


def consolidation_prefix(gpu, kernel, box_blocks, interval, safety=1.2):
    out, err = C.c_int64(), C.create_string_buffer(1024)
    _chk(lib().msref_consolidation_prefix(_j(gpu), _j(kernel), (C.c_int64 * max(1, len(box_blocks)))(*box_blocks),
                                          len(box_blocks), interval, safety, C.byref(out), err, 1024), err)
    return out.value


def percentile(samples, q):
    return lib().msref_percentile((C.c_int64 * max(1, len(samples)))(*samples), len(samples), q)


def generate_bursty_arrivals(rate, burstiness, horizon_ns, seed, dwell_ns=2_000_000_000):
    n, err = C.c_size_t(), C.create_string_buffer(1024)
    cap = int(rate * horizon_ns / 1e9 * 3 + 1024)
    while True:
        out = (C.c_int64 * cap)()
        rc = lib().msref_generate_bursty_arrivals(rate, burstiness, horizon_ns, seed & _U64, dwell_ns, out, cap,
                                                  C.byref(n), err, 1024)
        if rc == -4:
            cap = n.value
            continue
        _chk(rc, err)
        return list(out[: n.value])


def run_scenario(scenario, policy, ndjson=False, report=False, delays=False, options=None):
    flags = (1 if ndjson else 0) | (2 if report else 0) | (4 if delays else 0)
    out, err = C.c_void_p(), C.create_string_buffer(4096)
    L = lib()
    opts = json.dumps(options).encode() if options else None
    _chk(L.msref_replay_run_opts(_j(scenario), policy.encode(), opts, flags, C.byref(out), err, 4096), err)
    s = C.cast(out, C.c_char_p).value.decode()
    L.msref_free(out)
    return json.loads(s)


def parallel_runs(scenario, policy, n_threads):
    out, err = (C.c_double * 2)(), C.create_string_buffer(4096)
    _chk(lib().msref_parallel_runs(_j(scenario), policy.encode(), n_threads, out, err, 4096), err)
    return {"wall_s": out[0], "timeline_events": out[1]}
