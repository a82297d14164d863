"""On-B200 kernel profiler -> reference KernelSpec.

The paper profiles each LP kernel once and feeds the measurements to the split-plan search
(PAPER.md:628-630).  The reference consumes such a profile as `KernelSpec.measured_time`
— (n_blocks, time) rows interpolated piecewise-linearly by the execution oracle
(engine.hpp:461-481) that `find_optimal_split` searches (splitter.hpp:141-207).  This
module closes that loop on B200: it times a registered persistent LP kernel over tile
prefixes [0, n) with CUDA events (ms_lp_time_range), and emits a KernelSpec in the
reference scenario schema (scenario_io.hpp:128-200) whose grid is the tile space, whose
capacity (Eq. 1, exec_model.hpp:17-35) equals the kernel's resident CTAs, and whose
measured_time rows are the timings — ready for `microslice.find_optimal_split` and for the
replay engine.
"""
from __future__ import annotations

import math

from . import microslice as M
from .device import Device, LpKernel


def _dur(ns: int) -> dict:
    return {"value": int(ns), "unit": "ns"}


def sweep_points(total: int, per_wave: int) -> list[int]:
    """Tile counts to time: half a wave, 1, 2, 4, ... waves, and the whole range."""
    pts = {max(1, per_wave // 2), min(total, per_wave)}
    w = 2
    while w * per_wave < total:
        pts.add(w * per_wave)
        w *= 2
    pts.add(total)
    return sorted(p for p in pts if 1 <= p <= total)


def profile_lp_kernel(dev: Device, k: LpKernel, name: str, resident: int, tile_bytes: float,
                      reps: int = 3, points: list[int] | None = None) -> dict:
    """Time kernel `k` over tile prefixes and return a reference-schema KernelSpec.

    resident   : CTAs (= tiles in flight) the persistent kernel keeps on the GPU, i.e. the
                 Eq. 1 capacity the spec must reproduce (tpb 256, occupancy resident/8/SMs)
    tile_bytes : compulsory HBM bytes per tile (bw_demand_per_block = bytes / tile time)
    """
    pts = points or sweep_points(k.total_tiles, resident)
    rows = []
    for n in pts:
        ms = dev.lp_time_range(k, 0, n, reps)
        rows.append((n, int(round(ms * 1e6))))
    return kernel_spec(name, k.total_tiles, resident, dev.info["sm_count"], tile_bytes, rows)


def kernel_spec(name: str, total: int, resident: int, sms: int, tile_bytes: float, rows: list) -> dict:
    """Reference-schema KernelSpec from measured (n_tiles, ns) rows (the last row = the
    whole tile space)."""
    full_ns = rows[-1][1]
    waves = math.ceil(total / resident)
    tile_ns = max(1, full_ns // waves)
    per_sm = max(1, round(resident / sms))  # whole CTAs per SM (Eq. 1 floors o * 2048 / 256)
    return {
        "name": name,
        "grid": [int(total), 1, 1],
        "threads_per_block": 256,
        "occupancy": per_sm / 8.0,  # Eq. 1 (PerSmFloor): n_sm * floor(o * 2048 / 256) = n_sm * per_sm
        "block_time": {"dist": "point", "value": _dur(tile_ns)},
        "bw_demand_per_block": float(tile_bytes) / (tile_ns * 1e-9),
        "splittable": True,
        "measured_time": [{"n_blocks": int(n), "time": _dur(t)} for n, t in rows],
    }


def split_plan(gpu: dict, spec: dict, cap_ns: int = 400_000) -> dict:
    """Split plan of a profiled kernel (reference find_optimal_split over the measured
    oracle)."""
    return M.find_optimal_split(gpu, spec, cap_ns=cap_ns)
