"""Randomised scenario generator for the differential replay-parity tests.

Draws every knob the reference engine branches on: multi-dimensional grids, Eq. 1
occupancy / per-SM vs global floor, point / uniform / empirical / default block-time
CDFs, saturating HBM demand, splittable flags, measured_time oracles, repeats, hint
positions, contended hints, several HP and LP tasks, tiny resync_every, slice caps,
square tiling, consolidation on/off, REEF queue caps and eviction costs.
"""
from __future__ import annotations

import random


def _dur(ns):
    return {"value": int(ns), "unit": "ns"}


def _dist(rng: random.Random, lo_us=2, hi_us=120):
    k = rng.random()
    if k < 0.35:
        return {"dist": "point", "value": _dur(rng.randint(lo_us * 1000, hi_us * 1000))}
    if k < 0.7:
        a = rng.randint(lo_us * 1000, hi_us * 1000)
        return {"dist": "uniform", "lo": _dur(a), "hi": _dur(a + rng.randint(0, hi_us * 1000))}
    if k < 0.85:
        return {"dist": "default_cdf"}
    n = rng.randint(2, 5)
    vals = sorted(rng.randint(lo_us * 1000, hi_us * 4000) for _ in range(n))
    cums = sorted(rng.random() for _ in range(n - 2))
    pts = [{"t": _dur(v), "cdf": c} for v, c in zip(vals, [0.0] + cums + [1.0])]
    return {"dist": "empirical", "points": pts}


def random_scenario(seed: int, horizon_ms: float | None = None) -> dict:
    rng = random.Random(seed)
    n_sm = rng.choice([2, 4, 8, 16, 108, 148])
    smt = rng.choice([1024, 2048])
    gpu = {"n_sm": n_sm, "sm_max_threads": smt, "hbm_bandwidth": rng.choice([1e11, 2e12, 6.5157e12]),
           "launch_overhead": _dur(rng.randint(1000, 9000)), "sync_overhead": _dur(rng.randint(1000, 7000))}
    kernels = []
    for i in range(rng.randint(2, 6)):
        tpb = rng.choice([32, 64, 128, 256, 512, 1024])
        occ = rng.choice([1.0, 0.5, 0.25, 0.125, 0.75])
        while occ * smt < tpb:
            occ = min(1.0, occ * 2)
            if occ * smt < tpb:
                tpb //= 2
        dims = rng.choice([1, 2, 3])
        grid = [rng.randint(1, 64), rng.randint(1, 16) if dims > 1 else 1, rng.randint(1, 4) if dims > 2 else 1]
        k = {"name": f"k{i}", "grid": grid, "threads_per_block": tpb, "occupancy": occ,
             "block_time": _dist(rng), "bw_demand_per_block": rng.choice([0.0, 0.0, 1e8, 5e9, 5e10]),
             "splittable": rng.random() < 0.85}
        if rng.random() < 0.2:
            rows = sorted({rng.randint(1, 4096) for _ in range(rng.randint(1, 4))})
            k["measured_time"] = [{"n_blocks": r, "time": _dur(rng.randint(1000, 400000))} for r in rows]
        if rng.random() < 0.1 and grid[2] == 1:
            s = rng.choice([2, 4, 8, 16])
            k["grid"] = [s, s, 1]
        kernels.append(k)
    names = [k["name"] for k in kernels]
    horizon = horizon_ms if horizon_ms is not None else rng.choice([3, 8, 20, 40])
    tasks, traces = [], []
    for h in range(rng.choice([0, 1, 1, 1, 2])):
        seq = [{"kernel": rng.choice(names), "repeat": rng.randint(1, 3)} for _ in range(rng.randint(1, 4))]
        n_exp = sum(s["repeat"] for s in seq)
        hints = []
        for _ in range(rng.choice([0, 1, 1, 2, 3])):
            hints.append({"kind": rng.choice(["mem_sync", "inter_gpu_comm", "cpu_bound"]),
                          "pattern": rng.sample(["cudaMemcpyAsync", "cudaStreamSynchronize", "ncclAllReduce",
                                                 "cpu"], rng.randint(1, 2)),
                          "duration": _dist(rng, 5, 600), "position": rng.choice([-1, 0, rng.randint(0, n_exp)]),
                          "contended": rng.random() < 0.25})
        tname = f"tr{h}"
        tasks.append({"name": f"hp{h}", "priority": "high", "kind": "serving", "trace": tname, "kernels": seq,
                      "bubble_hints": hints})
        if rng.random() < 0.5:
            t, arr = 0, []
            for _ in range(rng.randint(1, 60)):
                t += rng.randint(1, int(horizon * 1e6 / 10) + 1)
                arr.append(t)
            tr = {"name": tname, "arrivals_ns": arr}
        else:
            tr = {"name": tname, "bursty": {"rate": rng.choice([400.0, 2000.0, 5000.0]),
                                            "burstiness": rng.choice([1.0, 2.0, 4.0])}}
        if rng.random() < 0.7:
            tr["iterations"] = rng.choice([{"dist": "point", "value": rng.randint(1, 9)},
                                           {"dist": "uniform", "lo": 1, "hi": rng.randint(1, 12)}])
        traces.append(tr)
    for l in range(rng.choice([0, 1, 1, 2, 3])):
        seq = [{"kernel": rng.choice(names), "repeat": rng.randint(1, 2)} for _ in range(rng.randint(1, 3))]
        tasks.append({"name": f"lp{l}", "priority": "low", "kind": "batch", "kernels": seq})
    rng.shuffle(tasks)
    sc = {"name": f"rand{seed}", "seed": rng.randint(1, 10**9), "horizon": _dur(int(horizon * 1e6)), "gpu": gpu,
          "kernels": kernels, "tasks": tasks, "traces": traces,
          "scheduler": {"threshold_ms": rng.choice([0.05, 0.2, 1.0, 2.0]), "ema_alpha": rng.choice([0.3, 0.5, 1.0]),
                        "ema_k": rng.randint(1, 8), "safety_factor": rng.choice([1.0, 1.2, 2.0]),
                        "resync_every": rng.choice([1, 2, 5, 64]), "slice_cap_us": rng.choice([20, 100, 400]),
                        "square_tiling": rng.random() < 0.3, "consolidation": rng.random() < 0.8},
          "reef": {"queue_cap": rng.randint(1, 4), "evict_cost_us": rng.choice([0, 1, 3])}}
    return sc


def random_memory_scenario(seed: int) -> dict:
    """random_scenario + the memory tier (engine.hpp:396-411, 1199-1276): task footprints
    that overflow a small local HBM, 0-3 NVLink peers with background load and limited
    free space, contention-first or round-robin eviction, 0-6 accesses per wave."""
    sc = random_scenario(seed)
    rng = random.Random(seed * 7919 + 13)
    n_peers = rng.choice([0, 1, 2, 3])
    sc["gpu"]["nvlink_peers"] = [
        {"peer_id": p + 1, "baseline_latency": _dur(rng.randint(500, 5000)),
         "bandwidth": rng.choice([5e10, 4.5e11, 9e11]),
         "background_load": rng.choice([0.0, 0.0, 1e11, 6e11, 2e12])} for p in range(n_peers)]
    if rng.random() < 0.5:
        sc["gpu"]["dram_latency_factor"] = rng.choice([1.0, 2.5, 8.0])
    hbm = rng.choice([0.05, 0.2, 1.0, 80.0])
    sc["memory"] = {"hbm_gb": hbm,
                    "peer_links": [{"free_gb": rng.choice([0.0, 0.01, 0.1, 5.0])} for _ in range(n_peers)],
                    "probe_mb": rng.choice([1.0, 4.0, 16.0]),
                    "score_threshold": rng.choice([1.05, 1.5, 3.0]),
                    "eviction": rng.choice(["contention_first", "round_robin"]),
                    "accesses_per_wave": rng.randint(0, 6)}
    if rng.random() < 0.5:
        sc["memory"]["dram_factor"] = rng.choice([1.0, 4.0, 10.0])
    for t in sc["tasks"]:
        if rng.random() < 0.85:
            limit = hbm * (0.6 if t["priority"] == "high" else 3.0)
            t["memory_footprint_gb"] = round(rng.uniform(0.0, limit), 4)
    return sc
