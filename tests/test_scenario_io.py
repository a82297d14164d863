"""Scenario wire format: parse / validate / round-trip with the
reference's semantics and error behaviour (ValidationError where-paths)."""
import copy

import pytest

from scenario_gen import random_scenario


def test_roundtrip_is_stable(ms):
    for seed in range(30):
        sc = random_scenario(seed)
        try:
            norm = ms.normalize_scenario(sc)
        except ms.ValidationError:
            continue
        assert ms.normalize_scenario(norm) == norm
        # a normalized scenario replays identically to the original
        assert ms.run_scenario(norm, "splitkernel")["timeline"] == ms.run_scenario(sc, "splitkernel")["timeline"]


@pytest.mark.parametrize("mutate,where", [
    (lambda s: s["tasks"].append({"name": "x", "priority": "low", "kind": "batch",
                                  "kernels": [{"kernel": "nope"}]}), "task.x"),
    (lambda s: s["gpu"].__setitem__("n_sm", 0), "gpu.n_sm"),
    (lambda s: s["kernels"][0].__setitem__("occupancy", 1.5), "kernel.occupancy"),
    (lambda s: s["gpu"].pop("sync_overhead"), "/gpu/sync_overhead"),
    (lambda s: s["kernels"][0]["block_time"].__setitem__("dist", "weird"), "/kernels/0/block_time/dist"),
    (lambda s: s.__setitem__("scheduler", {"ema_alpha": 0.0}), "scheduler.ema_alpha"),
    (lambda s: s["traces"][0].__setitem__("arrivals_ns", [5, 5]), "trace."),
])
def test_validation_errors_match_reference(ms, ref, mutate, where):
    from paper_2601_04071_b200 import scenarios as S
    sc = copy.deepcopy(S.config1(seed=1, horizon_s=0.01))
    sc["traces"][0] = {"name": "hp_trace", "arrivals_ns": [1000, 2000]}
    mutate(sc)
    with pytest.raises(ms.ValidationError) as mine:
        ms.run_scenario(sc, "splitkernel")
    with pytest.raises(ref.RefError) as theirs:
        ref.run_scenario(sc, "splitkernel")
    assert where in str(mine.value)
    assert str(mine.value) in str(theirs.value)


def test_durations_truncate_like_reference(ms, ref):
    from paper_2601_04071_b200 import scenarios as S
    sc = S.config1(seed=5, horizon_s=0.05)
    sc["scheduler"] = {"threshold_ms": 0.0019999999, "slice_cap_us": 123.9999}
    sc["gpu"]["launch_overhead"] = {"value": 7.6999, "unit": "us"}
    a = ms.run_scenario(sc, "splitkernel")
    b = ref.run_scenario(sc, "splitkernel")
    a.pop("wall_s"); a.pop("des_events"); b.pop("wall_s")
    assert a == b
