"""Why does split-kernel harvest less LP than the request-level kernel-boundary baseline on
configs 2/3 (HP = one-iteration requests, no hints)?  Per policy: LP tiles/s vs exclusive,
launches, preemptions, budget extensions, SLO attainment — plus split-kernel variants."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200 import live as L  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402

H = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
dev = Device(0)
out = {}
for cls in ("Config3", "Config2"):
    w = getattr(L, cls)(dev)
    c = w.calibrate()
    rate = w.hp_rate()
    sc = w.scenario(seed=11, horizon_s=H, rate=rate)
    gov = {"power_governor": True}
    ex = L.live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
    slo = ex["own_p99"]
    att = lambda rows: sum(1 for x in rows if x[4] and x[1] <= slo["ttft_ns"] and x[2] <= slo["tpot_ns"]) / len(rows)  # noqa
    exlp = L.live_run(dev, w.scenario(seed=11, horizon_s=2.0, rate=rate), "exclusive_lp", w.binding(),
                      w.options(timeline=False, **gov))
    res = {"calib": {k: v for k, v in c.items() if k not in ("lp_tile_ns",)}, "exclusive_att": att(ex["requests"]["rows"]),
           "exlp_tiles_per_s": exlp["lp"]["tiles_per_s"], "exlp_launches_per_s": exlp["lp"]["launches"] / 2.0}
    variants = [("reef_req", "reef_req", {}), ("splitkernel", "splitkernel", {}),
                ("splitkernel eager", "splitkernel", {"eager": True}),
                ("splitkernel ungoverned", "splitkernel", {"power_governor": False})]
    for label, pol, extra in variants:
        o = dict(gov)
        o.update(extra)
        r = L.live_run(dev, sc, pol, w.binding(), w.options(timeline=False, **o))
        lp = r["lp"]
        res[label] = {"att": att(r["requests"]["rows"]), "lp": lp["tiles_per_s"] / exlp["lp"]["tiles_per_s"],
                      "launches": lp["launches"], "preemptions": lp["preemptions"],
                      "extensions": lp["budget_extensions"], "parents": lp["parents_completed"],
                      "ring_p99_us": r["ring_to_first_hp_cta_all"].get("p99_ns", 0) / 1e3,
                      "lp_sms": (r.get("power_governor") or {}).get("mean_lp_sms"),
                      "lp_exit_p99_us": (lambda x: sorted(x)[max(0, -(-99 * len(x) // 100) - 1)] / 1e3 if x else None)(
                          r["samples"].get("preempt_flag_to_last_lp_exit", []))}
    out[cls] = res
    w.close()
print(json.dumps(out, indent=1))
dev.close()
