"""Config-4 live A/B (governed split-kernel): hint harvests sized from the hint's mean vs a
low quantile of its duration profile (option hint_quantile).  Two alternating rounds over
the same trace after one exclusive run (SLO)."""
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
sc = w.scenario(seed=11, horizon_s=horizon, rate=w.hp_rate(0.8))
ex = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
slo = {"ttft_ns": ex["own_p99"]["ttft_ns"], "tpot_ns": ex["own_p99"]["tpot_ns"]}
ex2 = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False, slo=slo))
exlp = live_run(dev, sc, "exclusive_lp", w.binding(), w.options(timeline=False, power_governor=True))
out = {"requests": ex["requests"]["n"], "exclusive_slo": ex2["slo_attainment"], "rows": []}
print(json.dumps(out), flush=True)
for rnd in range(2):
    for q in (None, 0.25, 0.1):
        o = {"power_governor": True}
        if q is not None:
            o["hint_quantile"] = q
        r = live_run(dev, sc, "splitkernel", w.binding(), w.options(timeline=False, slo=slo, **o))
        row = {"round": rnd, "hint_quantile": q, "slo": r["slo_attainment"],
               "lp_norm": r["lp"]["tiles_per_s"] / max(1e-9, exlp["lp"]["tiles_per_s"]),
               "preemptions": r["lp"]["preemptions"], "ring_p99_us": r["ring_to_first_hp_cta_all"].get("p99_ns", 0) / 1e3,
               "chain_p50_us": r["hp_chain_duration"].get("p50_ns", 0) / 1e3,
               "chain_p99_us": r["hp_chain_duration"].get("p99_ns", 0) / 1e3}
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
if len(sys.argv) > 2:
    Path(sys.argv[2]).write_text(json.dumps(out, indent=1) + "\n")
dev.close()
