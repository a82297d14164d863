"""A/B of the bs=1 decode chain's unit assignment (hp_gemv.cuh): MS_GEMV_DYNAMIC=1 (units
claimed per op by each CTA's producer) vs 0 (static round-robin plan).
  (1) chain alone: CUDA-event time per step (back-to-back direct launches);
  (2) config 4 live at 80% HP load, governed: SLO attainment vs exclusive, HP step p50 /
      p99 under co-location, LP throughput — alternating modes, same trace."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4, live_run  # noqa: E402

H = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
dev = Device(0)
w = Config4(dev)
w.calibrate()
out = {"alone_ms": {}}
for mode in ("1", "0", "1", "0"):
    os.environ["MS_GEMV_DYNAMIC"] = mode
    out["alone_ms"].setdefault(mode, []).append(min(dev.hp_time_chain(w.chain, 20) for _ in range(3)))
rate = w.hp_rate(0.8)
sc = w.scenario(seed=31, horizon_s=H, rate=rate)
ex = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
slo = {"ttft_ns": ex["own_p99"]["ttft_ns"], "tpot_ns": ex["own_p99"]["tpot_ns"]}


def att(rows):
    return sum(1 for x in rows if x[4] and x[1] <= slo["ttft_ns"] and x[2] <= slo["tpot_ns"]) / max(1, len(rows))


exlp = live_run(dev, w.scenario(seed=31, horizon_s=4.0, rate=rate), "exclusive_lp", w.binding(),
                w.options(timeline=False, power_governor=True))
out["exclusive"] = {"att": att(ex["requests"]["rows"]), "n": len(ex["requests"]["rows"]),
                    "step_p50_us": ex["hp_chain_duration"]["p50_ns"] / 1e3,
                    "step_p99_us": ex["hp_chain_duration"]["p99_ns"] / 1e3}
for rnd in range(2):
    for mode in ("1", "0"):
        os.environ["MS_GEMV_DYNAMIC"] = mode
        time.sleep(0.3)
        r = live_run(dev, sc, "splitkernel", w.binding(), w.options(timeline=False, power_governor=True))
        out[f"splitkernel dyn={mode} r{rnd}"] = {
            "att": att(r["requests"]["rows"]), "lp": r["lp"]["tiles_per_s"] / exlp["lp"]["tiles_per_s"],
            "step_p50_us": r["hp_chain_duration"]["p50_ns"] / 1e3, "step_p99_us": r["hp_chain_duration"]["p99_ns"] / 1e3,
            "ring_p99_us": r["ring_to_first_hp_cta_all"]["p99_ns"] / 1e3,
            "lp_exit_p99_us": r["preempt_flag_to_last_lp_exit"].get("p99_ns", 0) / 1e3}
print(json.dumps(out, indent=1))
dev.close()
