"""The oracle is pinned before it is trusted (task spec ③): the compiled reference
must reproduce the known answers published in SPEC.md / SURVEY.md §4, and the committed
golden fixtures (tests/golden/*.json, produced by tests/golden/make_golden.py from the
reference) must agree with the reference as built here."""
import json
from pathlib import Path

import pytest

GOLD = Path(__file__).resolve().parent / "golden"
KAT = json.loads((GOLD / "kat.json").read_text())

# Literal known answers with their published source.
PUBLISHED = {
    "splitmix64(0)": 16294208416658607535,
    "hash_str(hp)": 628894295916453061,
    "hash_combine(1,2)": 11812867941337419652,
    "eq1_a100": 864,                            # SPEC.md:135 (108 SM, 2048 thr, tpb 256, o 1.0)
    "eq1_one_block_per_sm": 108,
    "eq1_b200_persistent": 148,
    "default_cdf_mean": 67402,
    "default_cdf_s50": 57778,
    "default_cdf_s95": 201010,
    "ema_10_10_10_20ms": 13_000_000,
    "ema_empty": 2_000_000,
    "tick_77_7": 70_000,
    "consolidation_prefix_1ms": 10,
    "p99_99x10_20": 20_000_000,                 # SURVEY.md §4 / SPEC.md:673
    "poisson_60s_count": 621,                   # SURVEY.md §4 (+3.5% of 600)
}


def test_published_answers_in_golden():
    assert KAT["splitmix64"][0] == [0, PUBLISHED["splitmix64(0)"]]
    assert ["hp", PUBLISHED["hash_str(hp)"]] in KAT["hash_str"]
    assert [1, 2, PUBLISHED["hash_combine(1,2)"]] in KAT["hash_combine"]
    cc = [row[-1] for row in KAT["concurrent_capacity"]]
    assert cc[:3] == [PUBLISHED["eq1_a100"], PUBLISHED["eq1_one_block_per_sm"], PUBLISHED["eq1_b200_persistent"]]
    assert KAT["dist"]["default_cdf_mean"] == PUBLISHED["default_cdf_mean"]
    s = dict((u, v) for u, v in KAT["dist"]["default_cdf_samples"])
    assert s[0.5] == PUBLISHED["default_cdf_s50"] and s[0.95] == PUBLISHED["default_cdf_s95"]
    pi = {tuple(g): v for g, v in KAT["predict_interval"]}
    assert pi[(10_000_000, 10_000_000, 10_000_000, 20_000_000)] == PUBLISHED["ema_10_10_10_20ms"]
    assert pi[()] == PUBLISHED["ema_empty"]
    assert [77_000, 7_000, PUBLISHED["tick_77_7"]] in KAT["tick_interval"]
    assert KAT["consolidation_prefix"][0][-1] == PUBLISHED["consolidation_prefix_1ms"]
    assert KAT["percentile"][0][-1] == PUBLISHED["p99_99x10_20"]
    assert KAT["poisson_count"][0][-1] == PUBLISHED["poisson_60s_count"]
    # compute-bound split 864 blocks/slice, 77 us, 5 slices; on the
    # (64, 64) grid the boxes are 13 rows (832) with a last box of 12 rows (768);
    # memory-bound 440/slice; single block over the cap is uncappable.
    p = KAT["find_optimal_split"]
    assert (p[0][2]["blocks_per_slice"], p[0][2]["predicted_slice_time"], len(p[0][2]["slices"])) == (864, 77000, 5)
    assert [b[3] * b[4] for b in p[0][2]["slices"]] == [832, 832, 832, 832, 768]
    assert p[1][2]["blocks_per_slice"] == 440 and p[1][2]["memory_bound"]
    assert p[2][2]["uncappable"] and p[2][2]["blocks_per_slice"] == 1
    sb = {(tuple(g), n, sq): v for g, n, sq, v in KAT["slice_boxes"]}
    assert [b[3] * b[4] * b[5] for b in sb[((8, 1, 1), 3, False)]] == [3, 3, 2]
    assert KAT["consolidate"][0][-1] == [[0, 0, 0, 64, 64, 1]]           # 4 quadrants -> full box
    assert KAT["consolidate"][1][-1] == [[3, 0, 0, 5, 1, 1]]             # {3..7} -> offset 3, size 5


def test_reference_reproduces_golden(ref):
    """The reference as compiled here gives exactly the committed fixtures."""
    for x, v in KAT["splitmix64"]:
        assert ref.splitmix64(x) == v
    for s_, v in KAT["hash_str"]:
        assert ref.hash_str(s_) == v
    for a, b, v in KAT["hash_combine"]:
        assert ref.hash_combine(a, b) == v
    for g, k, r, v in KAT["concurrent_capacity"]:
        assert ref.concurrent_capacity(g, k, r) == v
    for g, k, n, v in KAT["exec_time_model"]:
        assert ref.exec_time_model(g, k, n) == v
    for g, n, sq, v in KAT["slice_boxes"]:
        assert [list(b) for b in ref.slice_boxes(g, n, sq)] == v
    for g, n, v in KAT["percentile"]:
        assert ref.percentile(g, n) == v
    for rate, b, h, seed, prefix in KAT["bursty_prefix"]:
        assert ref.generate_bursty_arrivals(rate, b, h, seed)[:20] == prefix


@pytest.mark.parametrize("field", ["splitmix64", "hash_str", "hash_combine", "u01_from_key"])
def test_product_keyed_rng_matches_golden(ms, field):
    for row in KAT[field]:
        *args, want = row
        assert getattr(ms, field)(*args) == want


def test_product_planning_matches_golden(ms):
    for g, k, r, v in KAT["concurrent_capacity"]:
        assert ms.concurrent_capacity(g, k, r) == v
    for g, k, n, v in KAT["exec_time_model"]:
        assert ms.exec_time_model(g, k, n) == v
    for g, k, plan in KAT["find_optimal_split"][:-1]:
        got = ms.find_optimal_split(g, k)
        got["slices"] = [list(b) for b in got["slices"]]
        assert got == plan
    g, k, plan = KAT["find_optimal_split"][-1]
    got = ms.find_optimal_split(g, k, square_tiling=True, cap_ns=10**9)
    got["slices"] = [list(b) for b in got["slices"]]
    assert got == plan
    for g, n, sq, v in KAT["slice_boxes"]:
        assert [list(b) for b in ms.slice_boxes(g, n, sq)] == v
    for g, pend, v in KAT["consolidate"]:
        assert [list(b) for b in ms.consolidate(g, pend)] == v
    for gaps, v in KAT["predict_interval"]:
        assert ms.predict_interval(gaps) == v
    for p, l, v in KAT["tick_interval"]:
        assert ms.tick_interval(p, l) == v
    for g, k, blocks, interval, safety, v in KAT["consolidation_prefix"]:
        assert ms.consolidation_prefix(g, k, blocks, interval, safety) == v
    for s_, q, v in KAT["percentile"]:
        assert ms.percentile(s_, q) == v
    for rate, b, h, seed, n in KAT["poisson_count"]:
        assert len(ms.generate_bursty_arrivals(rate, b, h, seed)) == n
    for rate, b, h, seed, prefix in KAT["bursty_prefix"]:
        assert ms.generate_bursty_arrivals(rate, b, h, seed)[:20] == prefix
    d = KAT["dist"]
    assert ms.dist_mean({"dist": "default_cdf"}) == d["default_cdf_mean"]
    for u, v in d["default_cdf_samples"]:
        assert ms.dist_sample({"dist": "default_cdf"}, [u]) == [v]
    uni = {"dist": "uniform", "lo": {"value": 500, "unit": "us"}, "hi": {"value": 1000, "unit": "us"}}
    for key, v in d["uniform_keyed"]:
        assert ms.dist_sample_keyed(uni, [key]) == [v]
