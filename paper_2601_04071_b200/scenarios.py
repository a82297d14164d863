"""BASELINE.json configs expressed as ScenarioSpec JSON.

Every config is a scenario in the reference's own schema (scenario_io.hpp:128-329) so
the reference CPU scheduler and this framework's replay engine consume the same bytes,
and the live B200 runtime is driven by the same task/kernel/trace description.

Replay GpuConfig = 148 SMs, 2048 threads/SM, HBM = MEASURED_PEAKS.json hbm_gbs, launch
and sync overheads measured on B200 (profiles/r01_latency_probe.txt: host launch ->
kernel start p50 7.68 us).  Kernel specs are calibrated from the sm_100a tenant kernels:
grid = tile count, tpb/occupancy chosen so Eq. 1 equals the persistent residency
(tpb 256, o = 0.125 -> 1 CTA/SM -> 148), block_time = measured per-tile time,
bw_demand_per_block = tile bytes / tile time.
"""
from __future__ import annotations

import copy
import json
from pathlib import Path

HBM_BPS = 6515.7e9  # MEASURED_PEAKS.json hbm_gbs
N_SM = 148

# Calibration of per-tile times on B200 (ns).  Defaults are roofline estimates; the
# bench overwrites them with measured values (profiles/).
DEFAULT_CALIB = {
    "launch_overhead_ns": 7680,     # profiles/r01_latency_probe.txt, launch p50
    "sync_overhead_ns": 5000,       # reference model default until measured
    "lp_gemm_tile_ns": 57000,       # 128x256x8192 bf16 tile at 1384.9 TFLOP/s / 148 SMs
    "lp_gemm_tile_bytes": (128 + 256) * 8192 * 2 + 128 * 256 * 2,
    "hp_gemm_tile_ns": 12000,       # 128x32 tile of 128x4096x4096, HBM-bound
    "hp_gemm_tile_bytes": (128 + 32) * 4096 * 2 + 128 * 32 * 2,
    "hp_ew_tile_ns": 2000,
    "hp_ew_tile_bytes": 128 * 4096 * 2 * 2 // 128,
    "lp_ew_tile_ns": 3000,
    "lp_ew_tile_bytes": 6 * 65536,
}


def _dur(ns: int) -> dict:
    return {"value": int(ns), "unit": "ns"}


def gpu_b200(calib: dict) -> dict:
    return {"n_sm": N_SM, "sm_max_threads": 2048, "hbm_bandwidth": HBM_BPS,
            "launch_overhead": _dur(calib["launch_overhead_ns"]),
            "sync_overhead": _dur(calib["sync_overhead_ns"])}


def _kernel(name, tiles, tile_ns, tile_bytes, splittable=True, per_sm=1, measured_time=None):
    # tpb 256 with occupancy per_sm/8 -> Eq. 1 = 148 * per_sm resident tiles.
    k = {"name": name, "grid": [int(tiles), 1, 1], "threads_per_block": 256,
         "occupancy": per_sm / 8.0, "block_time": {"dist": "point", "value": _dur(tile_ns)},
         "bw_demand_per_block": float(tile_bytes) / (tile_ns * 1e-9), "splittable": splittable}
    if measured_time:
        # on-B200 profile (profiler.profile_lp_kernel): the reference's measured execution
        # oracle (engine.hpp:461-481) for the split plan instead of the wave model
        k["measured_time"] = measured_time
    return k


def _lp_gemm_kernel(c: dict) -> dict:
    """The LP 8192^3 GEMM.  On CTA pairs (calib lp_gemm_tile_ctas = 2, 256 x 512 tiles) a
    tile holds two SMs for its tile time T: modelled as one block per SM whose block time is
    2 T (Eq. 1 capacity 148 x 1/(2T) = 74 tiles per T, the pair grid's real rate)."""
    ctas = int(c.get("lp_gemm_tile_ctas", 1))
    tile_bytes = c["lp_gemm_tile_bytes"] if ctas == 1 else (256 + 512) * 8192 * 2 + 256 * 512 * 2
    return _kernel("lp_gemm_8192", c.get("lp_gemm_tiles", 2048), c["lp_gemm_tile_ns"] * ctas, tile_bytes,
                   measured_time=c.get("lp_gemm_measured_time"))


def config1(seed: int = 1, horizon_s: float = 10.0, calib: dict | None = None, rate: float = 50.0) -> dict:
    """Config 1: HP small-GEMM-chain inference (Poisson) + LP batch GEMM loop."""
    c = dict(DEFAULT_CALIB, **(calib or {}))
    return {
        "name": "cfg1_gemm_chain_vs_gemm_loop",
        "seed": seed,
        "horizon": _dur(int(horizon_s * 1e9)),
        "gpu": gpu_b200(c),
        "kernels": [
            _kernel("hp_gemm_128x4096x4096", 128, c["hp_gemm_tile_ns"], c["hp_gemm_tile_bytes"], False),
            _kernel("hp_bias_gelu", 128, c["hp_ew_tile_ns"], c["hp_ew_tile_bytes"], False),
            _lp_gemm_kernel(c),
        ],
        "tasks": [
            {"name": "hp_infer", "priority": "high", "kind": "serving", "trace": "hp_trace",
             "kernels": [{"kernel": "hp_gemm_128x4096x4096", "repeat": 4}, {"kernel": "hp_bias_gelu"}],
             "bubble_hints": [{"kind": "mem_sync", "pattern": ["cudaMemcpyAsync", "cudaStreamSynchronize"],
                               "duration": {"dist": "uniform", "lo": _dur(500_000), "hi": _dur(1_000_000)},
                               "position": -1}]},
            {"name": "lp_train", "priority": "low", "kind": "batch", "kernels": [{"kernel": "lp_gemm_8192"}]},
        ],
        "traces": [{"name": "hp_trace", "bursty": {"rate": rate, "burstiness": 1.0},
                    "iterations": {"dist": "point", "value": 8}}],
    }


def config4(seed: int = 1, horizon_s: float = 10.0, calib: dict | None = None, rate: float = 20.0,
            threshold_ms: float | None = None) -> dict:
    """Config 4: Llama-style 1B decode HP (bs=1) + LP GEMM training + LP HBM streamer.
    `threshold_ms`: the scheduler's large-bubble threshold (scheduler.threshold_ms; None =
    the reference default, 2 ms)."""
    c = dict(DEFAULT_CALIB, **(calib or {}))
    sc = {
        "name": "cfg4_decode_vs_gemm_and_stream",
        "seed": seed,
        "horizon": _dur(int(horizon_s * 1e9)),
        "gpu": gpu_b200(c),
        "kernels": [
            _kernel("hp_decode_layer", 148, c.get("hp_layer_ns", 20_000), 148 * 1024 * 1024 // 148, False),
            _kernel("hp_lm_head", 148, c.get("hp_lm_head_ns", 40_000), 2048 * 128256 * 2 // 148, False),
            _lp_gemm_kernel(c),
            _kernel("lp_axpy_1g", c.get("lp_ew_tiles", 16384), c["lp_ew_tile_ns"], c["lp_ew_tile_bytes"], per_sm=4,
                    measured_time=c.get("lp_ew_measured_time")),
        ],
        "tasks": [
            {"name": "hp_decode", "priority": "high", "kind": "serving", "trace": "hp_trace",
             "kernels": [{"kernel": "hp_decode_layer", "repeat": 16}, {"kernel": "hp_lm_head"}],
             "bubble_hints": [{"kind": "cpu_bound", "pattern": ["sampling", "detokenize"],
                               "duration": {"dist": "uniform", "lo": _dur(100_000), "hi": _dur(500_000)},
                               "position": -1}]},
            {"name": "lp_gemm", "priority": "low", "kind": "batch", "kernels": [{"kernel": "lp_gemm_8192"}]},
            {"name": "lp_stream", "priority": "low", "kind": "batch", "kernels": [{"kernel": "lp_axpy_1g"}]},
        ],
        "traces": [{"name": "hp_trace", "bursty": {"rate": rate, "burstiness": 1.0},
                    "iterations": {"dist": "uniform", "lo": 32, "hi": 128}}],
    }
    if threshold_ms is not None:
        sc["scheduler"] = {"threshold_ms": threshold_ms}
    return sc


def config_memory(seed: int = 1, horizon_s: float = 10.0, calib: dict | None = None, rate: float = 20.0,
                  hp_gb: float = 60.0, lp_gb: tuple = (90.0, 60.0), hbm_gb: float = 180.0,
                  peer_free_gb: tuple = (40.0,) * 7, peer_load: tuple = (6e11, 0, 0, 3e11, 0, 0, 0),
                  eviction: str = "contention_first", accesses_per_wave: int = 4) -> dict:
    """Memory-intensive case on one B200 of an
    HGX node: config 4's tenants with footprints that overflow the 180 GB HBM (HP 60 GB
    pinned local; LP 150 GB, ~30 GB of it spilled), 7 NVLink-5 peers behind NVSwitch
    (900 GB/s each way, ~2 us zero-load latency), two of them carrying background traffic,
    DRAM as the last tier.  LP waves pay for their off-device chunks (engine.hpp:1199-1229);
    contention-first eviction steers spills away from the loaded links."""
    sc = config4(seed, horizon_s, calib, rate)
    sc["name"] = f"memory_{eviction}"
    sc["gpu"]["nvlink_peers"] = [{"peer_id": i + 1, "baseline_latency": _dur(2000), "bandwidth": 900e9,
                                  "background_load": float(peer_load[i])} for i in range(len(peer_free_gb))]
    sc["memory"] = {"hbm_gb": hbm_gb, "peer_links": [{"free_gb": g} for g in peer_free_gb],
                    "probe_mb": 4.0, "score_threshold": 1.5, "eviction": eviction,
                    "accesses_per_wave": accesses_per_wave}
    for t in sc["tasks"]:
        t["memory_footprint_gb"] = hp_gb if t["priority"] == "high" else lp_gb[0 if t["name"] == "lp_gemm" else 1]
    return sc


CONFIGS = {"cfg1": config1, "cfg4": config4, "memory": config_memory}


def with_seed(sc: dict, seed: int) -> dict:
    s = copy.deepcopy(sc)
    s["seed"] = seed
    return s


def dumps(sc: dict) -> str:
    return json.dumps(sc, sort_keys=True)


def save(sc: dict, path: str | Path) -> None:
    Path(path).write_text(json.dumps(sc, indent=2, sort_keys=True) + "\n")


def train_infer(name: str, seed: int, horizon_s: float, hp_task: str, hp_ops: int, hp_chain_ns: int, lp_task: str,
                lp_specs: list, lp_sequence: list, rate: float, threshold_ms: float = 0.5,
                calib: dict | None = None) -> dict:
    """Configs 2 / 3 (ResNet-50, BERT-base): one HP serving task whose request is ONE
    iteration of `hp_ops` chain kernels (point block time = measured chain time / ops, one
    wave each), Poisson arrivals at `rate`; one LP batch task whose kernel sequence is the
    training step (lp_sequence = [(kernel, repeat)], specs from TrainStepLP.kernel_specs)."""
    c = dict(DEFAULT_CALIB, **(calib or {}))
    op_ns = max(1000, hp_chain_ns // max(1, hp_ops))
    hp_kernel = _kernel(f"{hp_task}_op", N_SM, op_ns, 1 << 20, False)
    return {
        "name": name,
        "seed": seed,
        "horizon": _dur(int(horizon_s * 1e9)),
        "gpu": gpu_b200(c),
        "scheduler": {"threshold_ms": threshold_ms},
        "kernels": [hp_kernel] + list(lp_specs),
        "tasks": [
            {"name": hp_task, "priority": "high", "kind": "serving", "trace": "hp_trace",
             "kernels": [{"kernel": f"{hp_task}_op", "repeat": int(hp_ops)}], "bubble_hints": []},
            {"name": lp_task, "priority": "low", "kind": "batch",
             "kernels": [{"kernel": k, "repeat": int(r)} for k, r in lp_sequence]},
        ],
        "traces": [{"name": "hp_trace", "bursty": {"rate": rate, "burstiness": 1.0},
                    "iterations": {"dist": "point", "value": 1}}],
    }
