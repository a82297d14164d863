"""Regenerate the golden fixtures from the compiled REFERENCE (oracle/_ref/libmsref.so).

Run in the build container (needs /root/reference at build time):
    make -C oracle && python tests/golden/make_golden.py
Writes tests/golden/kat.json (known answers: the SURVEY.md §4 / SPEC.md examples, checked
against the reference itself) and tests/golden/replay_digests.json (decision-log digests of
the BASELINE configs and a randomised corpus, per policy), so parity can be asserted on
machines without the reference tree.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import ref as R  # noqa: E402
from paper_2601_04071_b200 import scenarios as S  # noqa: E402
from scenario_gen import random_memory_scenario, random_scenario  # noqa: E402

GPU_A100 = {"n_sm": 108, "sm_max_threads": 2048, "hbm_bandwidth": 2e12,
            "launch_overhead": {"value": 7, "unit": "us"}, "sync_overhead": {"value": 5, "unit": "us"}}
GPU_B200 = {"n_sm": 148, "sm_max_threads": 2048, "hbm_bandwidth": 6.5157e12,
            "launch_overhead": {"value": 7, "unit": "us"}, "sync_overhead": {"value": 5, "unit": "us"}}


def kernel(name, grid, tpb=256, occ=1.0, block_us=77, bw=0.0, **kw):
    k = {"name": name, "grid": grid, "threads_per_block": tpb, "occupancy": occ,
         "block_time": {"dist": "point", "value": {"value": block_us, "unit": "us"}}, "bw_demand_per_block": bw}
    k.update(kw)
    return k


def kats() -> dict:
    k = {}
    k["splitmix64"] = [[x, R.splitmix64(x)] for x in (0, 1, 2, 12345, 2**63, 2**64 - 1)]
    k["hash_str"] = [[s, R.hash_str(s)] for s in ("", "hp", "lp_train", "hp_infer#hint")]
    k["hash_combine"] = [[a, b, R.hash_combine(a, b)] for a, b in ((1, 2), (0, 0), (7, 2**40), (2**64 - 1, 3))]
    k["u01_from_key"] = [[x, R.u01_from_key(x)] for x in (0, 1, 99, 2**63)]
    # Eq. 1
    k["concurrent_capacity"] = [
        [GPU_A100, kernel("g", [64, 64, 1]), 0, R.concurrent_capacity(GPU_A100, kernel("g", [64, 64, 1]))],
        [GPU_A100, kernel("one", [8, 1, 1], tpb=2048), 0, R.concurrent_capacity(GPU_A100, kernel("one", [8, 1, 1], tpb=2048))],
        [GPU_B200, kernel("p", [2048, 1, 1], occ=0.125), 0, R.concurrent_capacity(GPU_B200, kernel("p", [2048, 1, 1], occ=0.125))],
        [GPU_A100, kernel("q", [9, 1, 1], tpb=384, occ=0.4), 1, R.concurrent_capacity(GPU_A100, kernel("q", [9, 1, 1], tpb=384, occ=0.4), 1)],
    ]
    # exec_time_model: single wave, two waves, memory-bound plateau
    cb = kernel("cb", [864, 1, 1])
    mb = kernel("mb", [4096, 1, 1], bw=2 * 2e12 / 864)
    k["exec_time_model"] = [[GPU_A100, kk, n, R.exec_time_model(GPU_A100, kk, n)]
                            for kk, n in ((cb, 1), (cb, 864), (cb, 1728), (mb, 864), (mb, 432), (mb, 216))]
    # split plans
    plans = []
    for gpu, kk in ((GPU_A100, kernel("gemm", [64, 64, 1])), (GPU_A100, mb),
                    (GPU_A100, kernel("big", [16, 1, 1], block_us=500)),
                    (GPU_B200, kernel("lpg", [2048, 1, 1], occ=0.125, block_us=57)),
                    (GPU_B200, kernel("ew", [16384, 1, 1], occ=0.5, block_us=3, bw=6.5157e12 / 400))):
        plans.append([gpu, kk, R.find_optimal_split(gpu, kk)])
    plans.append([GPU_A100, kernel("sq", [64, 64, 1]), R.find_optimal_split(GPU_A100, kernel("sq", [64, 64, 1]),
                                                                            square_tiling=True, cap_ns=10**9)])
    k["find_optimal_split"] = plans
    k["slice_boxes"] = [[g, n, sq, R.slice_boxes(g, n, sq)] for g, n, sq in
                        (([8, 1, 1], 3, False), ([64, 64, 1], 1184, False), ([64, 64, 1], 864, False),
                         ([64, 64, 1], 1024, True), ([5, 3, 2], 7, False), ([5, 3, 2], 20, False))]
    quads = R.slice_boxes([64, 64, 1], 1024, True)
    k["consolidate"] = [[[64, 64, 1], quads, R.consolidate([64, 64, 1], quads)],
                        [[16, 1, 1], [[3, 0, 0, 2, 1, 1], [5, 0, 0, 3, 1, 1]],
                         R.consolidate([16, 1, 1], [[3, 0, 0, 2, 1, 1], [5, 0, 0, 3, 1, 1]])]]
    k["predict_interval"] = [[g, R.predict_interval(g)] for g in
                             ([], [10_000_000, 10_000_000, 10_000_000, 20_000_000], list(range(1, 20)))]
    k["tick_interval"] = [[p, l, R.tick_interval(p, l)] for p, l in ((77_000, 7_000), (5_000, 7_000), (7_000, 7_000))]
    k["consolidation_prefix"] = [[GPU_A100, cb, [864] * 12, 1_000_000, 1.2,
                                  R.consolidation_prefix(GPU_A100, cb, [864] * 12, 1_000_000, 1.2)]]
    k["percentile"] = [[[10_000_000] * 99 + [20_000_000], 0.99, R.percentile([10_000_000] * 99 + [20_000_000], 0.99)],
                       [[5, 1, 4, 2, 3], 0.5, R.percentile([5, 1, 4, 2, 3], 0.5)], [[], 0.99, 0]]
    k["poisson_count"] = [[10.0, 1.0, 60 * 10**9, 42, len(R.generate_bursty_arrivals(10.0, 1.0, 60 * 10**9, 42))]]
    k["bursty_prefix"] = [[50.0, 2.0, 10**9, 7, R.generate_bursty_arrivals(50.0, 2.0, 10**9, 7)[:20]]]
    dcdf = {"dist": "default_cdf"}
    k["dist"] = {"default_cdf_mean": R.dist_mean(dcdf),
                 "default_cdf_samples": [[u, R.dist_sample(dcdf, [u])[0]] for u in (0.0, 0.5, 0.9, 0.95, 0.999999)],
                 "uniform_keyed": [[x, R.dist_sample_keyed({"dist": "uniform", "lo": {"value": 500, "unit": "us"},
                                                             "hi": {"value": 1000, "unit": "us"}}, [x])[0]]
                                   for x in (1, 2, 3, 2**50)]}
    return k


def digests() -> dict:
    out = {}
    cases = {"cfg1_seed1_0p5s": S.config1(seed=1, horizon_s=0.5), "cfg1_seed2_0p5s": S.config1(seed=2, horizon_s=0.5),
             "cfg4_seed1_0p2s": S.config4(seed=1, horizon_s=0.2)}
    for seed in range(40):
        cases[f"rand{seed}"] = random_scenario(1000 + seed)
    for seed in range(12):
        cases[f"mem{seed}"] = random_memory_scenario(2000 + seed)
    for ev in ("contention_first", "round_robin"):
        cases[f"memory_{ev}_0p3s"] = S.config_memory(seed=1, horizon_s=0.3, eviction=ev)
    # configs 2 / 3 (ResNet-50, BERT-base): training-step LP tasks, device-free specs
    from paper_2601_04071_b200 import tenants as TN
    for nm, g, n_par, mode, ops, rate in (("cfg2", TN.resnet50_train_gemms(64), TN.RESNET50_PARAMS, 1, 160, 200.0),
                                          ("cfg3", TN.bert_train_gemms(32), TN.BERT_PARAMS, 0, 96, 100.0)):
        specs, seq = TN.step_specs(nm, g, n_par, mode)
        for seed in (1, 2):
            cases[f"{nm}_seed{seed}_0p3s"] = S.train_infer(nm, seed=seed, horizon_s=0.3, hp_task=f"hp_{nm}", hp_ops=ops,
                                                          hp_chain_ns=900_000, lp_task=f"lp_{nm}", lp_specs=specs,
                                                          lp_sequence=seq, rate=rate)
    for name, sc in cases.items():
        out[name] = {"scenario": sc, "policies": {}}
        for pol in ("exclusive", "exclusive_lp", "splitkernel", "spatial", "reef"):
            try:
                d = R.run_scenario(sc, pol)
                d.pop("wall_s", None)
            except R.RefError as e:
                d = {"error_rc": e.rc, "error": str(e)}
            out[name]["policies"][pol] = d
    return out


if __name__ == "__main__":
    here = Path(__file__).resolve().parent
    (here / "kat.json").write_text(json.dumps(kats(), indent=1) + "\n")
    (here / "replay_digests.json").write_text(json.dumps(digests(), indent=1, sort_keys=True) + "\n")
    print("wrote", here / "kat.json", here / "replay_digests.json")
