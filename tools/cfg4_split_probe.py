"""Config 4 with the LP GEMM cut into k-slices (split 1 / 2 / 4): LP GEMM alone, and live
at 80% HP load under the governor — split-kernel vs request-level kernel boundary (SLO vs
exclusive, LP vs exclusive, ratio), same trace."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4, live_run  # noqa: E402

H = float(sys.argv[1]) if len(sys.argv) > 1 else 12.0
dev = Device(0)
out = {}
for split in (1, 2, 4):
    w = Config4(dev, lp_split=split)
    c = w.calibrate()
    rate = w.hp_rate(0.8)
    sc = w.scenario(seed=43, horizon_s=H, rate=rate)
    gov = {"power_governor": True}
    ex = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
    slo = ex["own_p99"]
    att = lambda rows: sum(1 for x in rows if x[4] and x[1] <= slo["ttft_ns"] and x[2] <= slo["tpot_ns"]) / len(rows)  # noqa
    exlp = live_run(dev, w.scenario(seed=43, horizon_s=4.0, rate=rate), "exclusive_lp", w.binding(),
                    w.options(timeline=False, **gov))
    res = {"lp_gemm_ms": c["lp_gemm_ms"], "tflops": 2 * 8192 ** 3 / (c["lp_gemm_ms"] * 1e-3) / 1e12,
           "exclusive_att": att(ex["requests"]["rows"]), "n": len(ex["requests"]["rows"])}
    for pol in ("splitkernel", "reef_req"):
        time.sleep(0.3)
        r = live_run(dev, sc, pol, w.binding(), w.options(timeline=False, **gov))
        res[pol] = {"att": att(r["requests"]["rows"]), "lp": r["lp"]["tiles_per_s"] / exlp["lp"]["tiles_per_s"],
                    "lp_exit_p99_us": r["preempt_flag_to_last_lp_exit"].get("p99_ns", 0) / 1e3,
                    "ring_p99_us": r["ring_to_first_hp_cta_all"].get("p99_ns", 0) / 1e3,
                    "step_p99_us": r["hp_chain_duration"]["p99_ns"] / 1e3}
    res["ratio"] = res["splitkernel"]["lp"] / max(1e-9, res["reef_req"]["lp"])
    out[split] = res
    print(json.dumps({split: res}), flush=True)
print(json.dumps(out, indent=1))
dev.close()
