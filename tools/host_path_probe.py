"""Config-4 live: host-side HP path latencies per policy — chain done (device) -> the
scheduler saw it, and bubble-end timer lateness — next to SLO attainment and LP."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4, live_run  # noqa: E402

horizon = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
dev = Device(0)
w = Config4(dev)
w.calibrate()
sc = w.scenario(seed=13, horizon_s=horizon, rate=w.hp_rate(0.8))
ex = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
slo = {"ttft_ns": ex["own_p99"]["ttft_ns"], "tpot_ns": ex["own_p99"]["tpot_ns"]}
out = []
for pol, o in (("exclusive", {}), ("splitkernel", {"power_governor": True}), ("splitkernel", {"lp_max_sms": 40}),
               ("reef_req", {"power_governor": True})):
    r = live_run(dev, sc, pol, w.binding(), w.options(timeline=False, slo=slo, **o))
    q = lambda k: (r.get(k) or {})  # noqa: E731
    row = {"policy": pol, "opts": o, "slo": r.get("slo_attainment"), "own_p99": r.get("own_p99"),
           "detect_lag": {m: q("hp_done_detect_lag").get(m) for m in ("p50_ns", "p90_ns", "p99_ns", "max_ns")},
           "timer_late": {m: q("bubble_timer_late").get(m) for m in ("p50_ns", "p90_ns", "p99_ns", "max_ns")},
           "ring_to_first": {m: q("ring_to_first_hp_cta_all").get(m) for m in ("p50_ns", "p99_ns")},
           "chain": {m: q("hp_chain_duration").get(m) for m in ("p50_ns", "p99_ns")}}
    out.append(row)
    print(json.dumps(row), flush=True)
if len(sys.argv) > 2:
    Path(sys.argv[2]).write_text(json.dumps(out, indent=1) + "\n")
dev.close()
