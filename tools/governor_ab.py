"""Config-4 live A/B (split-kernel): power-governor settings vs HP SLO attainment and LP.
Same trace for every variant, two alternating rounds after one exclusive run (SLO)."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4, live_run  # noqa: E402

horizon = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
dev = Device(0)
w = Config4(dev)
w.calibrate()
sc = w.scenario(seed=13, horizon_s=horizon, rate=w.hp_rate(0.8))
ex = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
slo = {"ttft_ns": ex["own_p99"]["ttft_ns"], "tpot_ns": ex["own_p99"]["tpot_ns"]}
ex2 = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False, slo=slo))
exlp = live_run(dev, sc, "exclusive_lp", w.binding(), w.options(timeline=False, power_governor=True))
out = {"requests": ex["requests"]["n"], "exclusive_slo": ex2["slo_attainment"], "rows": []}
print(json.dumps(out), flush=True)
variants = {"gov_default": {"power_governor": True},
            "gov_slack10": {"power_governor": True, "governor_slack_mhz": 10},
            "gov_min20": {"power_governor": True, "governor_min_sms": 20, "governor_slack_mhz": 10},
            "lp_max_40": {"lp_max_sms": 40}}
for rnd in range(2):
    for name, o in variants.items():
        r = live_run(dev, sc, "splitkernel", w.binding(), w.options(timeline=False, slo=slo, **o))
        row = {"round": rnd, "variant": name, "slo": r["slo_attainment"],
               "lp_norm": r["lp"]["tiles_per_s"] / max(1e-9, exlp["lp"]["tiles_per_s"]),
               "mean_lp_sms": (r.get("power_governor") or {}).get("mean_lp_sms"),
               "sm_mhz": (r.get("power_governor") or {}).get("mean_sm_mhz"),
               "ring_p99_us": r["ring_to_first_hp_cta_all"].get("p99_ns", 0) / 1e3,
               "chain_p50_us": r["hp_chain_duration"].get("p50_ns", 0) / 1e3,
               "chain_p99_us": r["hp_chain_duration"].get("p99_ns", 0) / 1e3}
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
    r = live_run(dev, sc, "reef_req", w.binding(), w.options(timeline=False, slo=slo, power_governor=True))
    out["rows"].append({"round": rnd, "variant": "reef_req_gov", "slo": r["slo_attainment"],
                        "lp_norm": r["lp"]["tiles_per_s"] / max(1e-9, exlp["lp"]["tiles_per_s"])})
    print(json.dumps(out["rows"][-1]), flush=True)
if len(sys.argv) > 2:
    Path(sys.argv[2]).write_text(json.dumps(out, indent=1) + "\n")
dev.close()
