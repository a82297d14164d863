"""Config 1: HP SLO attainment and LP throughput under split-kernel with LP's SM footprint
capped only inside HP requests (live option small_bubble_sms) vs uncapped vs governed, on
the same trace windows, interleaved (exclusive first in every window).  SLO = exclusive's
pooled p99 TTFT / TPOT."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, live_run  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 6
variants = [("uncapped", {}), ("in_request_74", {"small_bubble_sms": 74}), ("in_request_100", {"small_bubble_sms": 100}),
            ("in_request_50", {"small_bubble_sms": 50}), ("governed", {"power_governor": True})]
dev = Device(0)
w = Config1(dev)
w.calibrate(reps=3)
exlp = live_run(dev, w.scenario(seed=900, horizon_s=2.5), "exclusive_lp", w.binding(), w.options(timeline=False))
ex_rows, acc = [], {n: {"rows": [], "tiles": 0, "infl": []} for n, _ in variants}
for k in range(W):
    sc = w.scenario(seed=1000 + k, horizon_s=2.5)
    ex_rows += live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))["requests"]["rows"]
    for n, o in variants:
        r = live_run(dev, sc, "splitkernel", w.binding(), w.options(timeline=False, **o))
        acc[n]["rows"] += r["requests"]["rows"]
        acc[n]["tiles"] += r["lp"]["tiles_done"]
        acc[n]["infl"] += r["samples"]["preempt_ring_to_first_hp_cta_lp_in_flight"]


def p99(xs):
    s = sorted(xs)
    return s[min(len(s) - 1, int(0.99 * len(s)))] if s else None


slo = (p99([x[1] for x in ex_rows if x[4]]), p99([x[2] for x in ex_rows if x[4]]))
att = lambda rows: sum(1 for x in rows if x[4] and x[1] <= slo[0] and x[2] <= slo[1]) / max(1, len(rows))  # noqa
out = {"windows": W, "requests": len(ex_rows), "exclusive_att": round(att(ex_rows), 4)}
for n, _ in variants:
    a = acc[n]
    out[n] = {"att": round(att(a["rows"]), 4), "lp": round(a["tiles"] / (W * 2.5) / exlp["lp"]["tiles_per_s"], 4),
              "inflight_p99_us": (p99(a["infl"]) or 0) / 1e3}
print(json.dumps(out, indent=1))
dev.close()
