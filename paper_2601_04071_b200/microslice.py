"""Python view of the microslice scheduler API (names follow the reference's
namespace microslice, /root/reference/proj/include/microslice).  Every call goes
through libmicroslice.so's C-ABI (include/ms_replay.h); nothing is computed in Python.

Complex inputs (GpuConfig / KernelSpec / ScenarioSpec / DurationDist) are plain dicts
in the reference's scenario JSON schema (scenario_io.hpp:128-329).
"""
from __future__ import annotations

import ctypes as C
import json
from typing import Sequence

from . import _native as N

__all__ = [
    "splitmix64", "hash_combine", "hash_str", "u01_from_key", "dist_sample", "dist_sample_keyed",
    "dist_mean", "concurrent_capacity", "exec_time_model", "find_optimal_split", "slice_boxes",
    "consolidate", "predict_interval", "tick_interval", "consolidation_prefix", "percentile",
    "generate_bursty_arrivals", "run_scenario", "normalize_scenario", "ValidationError", "EngineError",
]

ValidationError = N.ValidationError
EngineError = N.EngineError
_U64 = (1 << 64) - 1


def _j(x) -> bytes:
    return (x if isinstance(x, str) else json.dumps(x)).encode()


def splitmix64(x: int) -> int:
    return N.core().ms_splitmix64(x & _U64)


def hash_combine(a: int, b: int) -> int:
    return N.core().ms_hash_combine(a & _U64, b & _U64)


def hash_str(s: str) -> int:
    b = s.encode()
    return N.core().ms_hash_str(b, len(b))


def u01_from_key(key: int) -> float:
    return N.core().ms_u01_from_key(key & _U64)


def dist_sample(dist: dict, us: Sequence[float]) -> list[int]:
    n = len(us)
    u = (C.c_double * n)(*us)
    out = (C.c_int64 * n)()
    err = N.errbuf()
    N.check(N.core().ms_dist_sample(_j(dist), u, n, out, err, len(err)), err)
    return list(out)


def dist_sample_keyed(dist: dict, keys: Sequence[int]) -> list[int]:
    n = len(keys)
    k = (C.c_uint64 * n)(*[x & _U64 for x in keys])
    out = (C.c_int64 * n)()
    err = N.errbuf()
    N.check(N.core().ms_dist_sample_keyed(_j(dist), k, n, out, err, len(err)), err)
    return list(out)


def dist_mean(dist: dict) -> int:
    out, err = C.c_int64(), N.errbuf()
    N.check(N.core().ms_dist_mean(_j(dist), C.byref(out), err, len(err)), err)
    return out.value


def concurrent_capacity(gpu: dict, kernel: dict, rounding: int = 0) -> int:
    out, err = C.c_int64(), N.errbuf()
    N.check(N.core().ms_concurrent_capacity(_j(gpu), _j(kernel), rounding, C.byref(out), err, len(err)), err)
    return out.value


def exec_time_model(gpu: dict, kernel: dict, n_blocks: int, load: float = 0.0, rounding: int = 0) -> int:
    out, err = C.c_int64(), N.errbuf()
    N.check(N.core().ms_exec_time_model(_j(gpu), _j(kernel), n_blocks, load, rounding, C.byref(out), err,
                                        len(err)), err)
    return out.value


def find_optimal_split(gpu: dict, kernel: dict, epsilon: float = 0.02, cap_ns: int = 400_000,
                       square_tiling: bool = False, rounding: int = 0) -> dict:
    plan, err = N.MsSplitPlan(), N.errbuf()
    lib = N.core()
    N.check(lib.ms_find_optimal_split(_j(gpu), _j(kernel), epsilon, cap_ns, int(square_tiling), rounding,
                                      C.byref(plan), None, 0, err, len(err)), err)
    boxes = (N.MsBox * max(1, plan.n_slices))()
    N.check(lib.ms_find_optimal_split(_j(gpu), _j(kernel), epsilon, cap_ns, int(square_tiling), rounding,
                                      C.byref(plan), boxes, plan.n_slices, err, len(err)), err)
    return {"blocks_per_slice": plan.blocks_per_slice, "predicted_slice_time": plan.predicted_slice_time_ns,
            "cap": plan.cap_ns, "memory_bound": bool(plan.memory_bound), "uncappable": bool(plan.uncappable),
            "slices": [boxes[i].astuple() for i in range(plan.n_slices)]}


def _boxes_call(fn, *args) -> list[tuple]:
    n = C.c_size_t()
    rc = fn(*args, None, 0, C.byref(n))
    if rc not in (N.MS_OK, N.MS_E_CAPACITY):
        N.check(rc)
    out = (N.MsBox * max(1, n.value))()
    N.check(fn(*args, out, n.value, C.byref(n)))
    return [out[i].astuple() for i in range(n.value)]


def slice_boxes(grid: Sequence[int], blocks_per_slice: int, square_tiling: bool = False) -> list[tuple]:
    gx, gy, gz = grid
    return _boxes_call(N.core().ms_slice_boxes, gx, gy, gz, blocks_per_slice, int(square_tiling))


def consolidate(grid: Sequence[int], pending: Sequence[Sequence[int]]) -> list[tuple]:
    gx, gy, gz = grid
    arr = (N.MsBox * max(1, len(pending)))(*[N.MsBox(*b) for b in pending])
    return _boxes_call(N.core().ms_consolidate, gx, gy, gz, arr, len(pending))


def predict_interval(gaps: Sequence[int], alpha: float = 0.3, k: int = 8, fallback: int = 2_000_000) -> int:
    arr = (C.c_int64 * max(1, len(gaps)))(*gaps)
    return N.core().ms_predict_interval(arr, len(gaps), alpha, k, fallback)


def tick_interval(predicted_slice_time: int, launch_overhead: int) -> int:
    return N.core().ms_tick_interval(predicted_slice_time, launch_overhead)


def consolidation_prefix(gpu: dict, kernel: dict, box_blocks: Sequence[int], predicted_interval: int,
                         safety_factor: float = 1.2) -> int:
    arr = (C.c_int64 * max(1, len(box_blocks)))(*box_blocks)
    out, err = C.c_int64(), N.errbuf()
    N.check(N.core().ms_consolidation_prefix(_j(gpu), _j(kernel), arr, len(box_blocks), predicted_interval,
                                             safety_factor, C.byref(out), err, len(err)), err)
    return out.value


def percentile(samples: Sequence[int], q: float) -> int:
    arr = (C.c_int64 * max(1, len(samples)))(*samples)
    return N.core().ms_percentile(arr, len(samples), q)


def generate_bursty_arrivals(rate: float, burstiness: float, horizon_ns: int, seed: int,
                             dwell_ns: int = 2_000_000_000) -> list[int]:
    lib, err, n = N.core(), N.errbuf(), C.c_size_t()
    cap = int(rate * horizon_ns / 1e9 * 3 + 1024)
    while True:
        out = (C.c_int64 * cap)()
        rc = lib.ms_generate_bursty_arrivals(rate, burstiness, horizon_ns, seed & _U64, dwell_ns, out, cap,
                                             C.byref(n), err, len(err))
        if rc == N.MS_E_CAPACITY:
            cap = n.value
            continue
        N.check(rc, err)
        return list(out[: n.value])


def run_scenario(scenario, policy: str, ndjson: bool = False, report: bool = False,
                 delays: bool = False, options: dict | None = None, rows: bool = False) -> dict:
    flags = (N.MS_RUN_NDJSON if ndjson else 0) | (N.MS_RUN_REPORT if report else 0) | \
            (N.MS_RUN_DELAYS if delays else 0) | (N.MS_RUN_ROWS if rows else 0)
    return N.replay_run(scenario, policy, flags, options)


def normalize_scenario(scenario) -> dict:
    lib, err, out = N.core(), N.errbuf(), C.c_void_p()
    N.check(lib.ms_scenario_normalize(_j(scenario), C.byref(out), err, len(err)), err)
    return json.loads(N.take_string(lib, out))
