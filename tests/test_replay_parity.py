"""Decision-log parity (BASELINE.json north_star): the B200 framework's scheduler core in
deterministic trace-replay mode must reproduce the reference CPU implementation's
admit / preempt / resume log byte-for-byte — every Timeline record, every RunArtifacts
vector and counter — for every in-scope policy.

* against committed golden digests (no reference needed): configs 1/4 + a random corpus
* differential, randomised, against the compiled reference (oracle/_ref)
"""
import json
from pathlib import Path

import pytest

from scenario_gen import random_memory_scenario, random_scenario

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "replay_digests.json").read_text())
POLICIES = ("exclusive", "exclusive_lp", "splitkernel", "spatial", "reef")


def _strip(d):
    d = dict(d)
    for k in ("wall_s", "des_events", "ndjson", "delays"):
        d.pop(k, None)
    return d


@pytest.mark.parametrize("case", sorted(GOLD))
def test_replay_matches_golden_digest(ms, case):
    sc = GOLD[case]["scenario"]
    for pol in POLICIES:
        want = GOLD[case]["policies"][pol]
        if "error_rc" in want:
            with pytest.raises((ms.ValidationError, ms.EngineError)):
                ms.run_scenario(sc, pol)
            continue
        assert _strip(ms.run_scenario(sc, pol)) == want, (case, pol)


@pytest.mark.parametrize("block", range(6))
def test_replay_differential_random(ms, ref, block):
    for seed in range(block * 60, block * 60 + 60):
        sc = random_scenario(seed)
        for pol in POLICIES:
            try:
                want = _strip(ref.run_scenario(sc, pol))
            except ref.RefError as e:
                with pytest.raises((ms.ValidationError, ms.EngineError)) as ei:
                    ms.run_scenario(sc, pol)
                assert str(ei.value) in str(e)
                continue
            assert _strip(ms.run_scenario(sc, pol)) == want, (seed, pol)


@pytest.mark.parametrize("block", range(3))
def test_replay_memory_tier_differential(ms, ref, block):
    """Memory tier (memory.hpp; engine.hpp:396-411, 798-801, 1199-1276): chunk placement,
    HP displacement errors, peer / DRAM faults, link congestion, ProbeTick cadence —
    NDJSON byte-equal with the compiled reference."""
    faults = 0
    for seed in range(block * 40, block * 40 + 40):
        sc = random_memory_scenario(seed)
        for pol in POLICIES:
            try:
                want = ref.run_scenario(sc, pol, ndjson=True)
            except ref.RefError as e:
                with pytest.raises((ms.ValidationError, ms.EngineError)) as ei:
                    ms.run_scenario(sc, pol)
                assert str(ei.value) in str(e)
                continue
            got = ms.run_scenario(sc, pol, ndjson=True)
            faults += want["ndjson"].count('"mem_fault"')
            assert got["ndjson"] == want["ndjson"], (seed, pol)
            assert _strip(got) == _strip(want), (seed, pol)
    assert faults > 0


def test_replay_ndjson_bytes_and_options(ms, ref):
    """Byte-level NDJSON equality plus EngineOptions (hint filter, global floor, sampling)."""
    for seed in (3, 17, 29, 41):
        sc = random_scenario(10_000 + seed)
        for opts in (None, {"global_floor": True}, {"hint_filter": ["cudaMemcpyAsync"]},
                     {"util_sample_period_ns": 37_000}):
            for pol in ("splitkernel", "exclusive_lp", "reef"):
                try:
                    want = ref.run_scenario(sc, pol, ndjson=True, options=opts)
                except ref.RefError:
                    continue
                got = ms.run_scenario(sc, pol, ndjson=True, options=opts)
                assert got["ndjson"] == want["ndjson"], (seed, opts, pol)
                assert _strip(got) == _strip(want)


def test_replay_reports_match(ms, ref):
    from paper_2601_04071_b200 import scenarios as S
    sc = S.config1(seed=3, horizon_s=2.5)
    a = ms.run_scenario(sc, "splitkernel", report=True, delays=True)
    b = ref.run_scenario(sc, "splitkernel", report=True, delays=True)
    assert a["report"] == b["report"]
    assert a["delays"] == b["delays"]


def test_replay_is_deterministic(ms):
    sc = random_scenario(77)
    assert _strip(ms.run_scenario(sc, "splitkernel")) == _strip(ms.run_scenario(sc, "splitkernel"))
