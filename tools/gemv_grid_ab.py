"""Decode chain (config 4) with a smaller GEMV grid (MS_GEMV_GRID, fixed at chain
registration): step time alone, and live at 80% HP load under the governor — SLO vs
exclusive, step p50 / p99, ring -> first HP CTA p99, LP throughput.  A chain of G < SMs-1
CTAs starts once G SMs are free instead of waiting for the last preempted LP CTA."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4, decode_step_ops, live_run  # noqa: E402

H = float(sys.argv[1]) if len(sys.argv) > 1 else 12.0
grids = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["147", "136", "124", "112"])]
dev = Device(0)
w = Config4(dev)
w.calibrate()
chains = {}
for g in grids:
    os.environ["MS_GEMV_GRID"] = str(g)
    chains[g] = dev.hp_register_chain(decode_step_ops(w.M, w.H, w.Q, w.F, w.V, w.LAYERS, w.bufs, w.weights, w.lm))
os.environ.pop("MS_GEMV_GRID")
out = {"alone_ms": {g: round(min(dev.hp_time_chain(c, 20) for _ in range(3)), 4) for g, c in chains.items()}}
rate = w.hp_rate(0.8)
sc = w.scenario(seed=41, horizon_s=H, rate=rate)
exlp = live_run(dev, w.scenario(seed=41, horizon_s=4.0, rate=rate), "exclusive_lp", w.binding(),
                w.options(timeline=False, power_governor=True))
for g, c in chains.items():
    b = w.binding()
    b["hp"]["hp_decode"] = [c]
    ex = live_run(dev, sc, "exclusive", b, w.options(timeline=False))
    slo = ex["own_p99"]
    att = lambda rows: sum(1 for x in rows if x[4] and x[1] <= slo["ttft_ns"] and x[2] <= slo["tpot_ns"]) / len(rows)  # noqa
    time.sleep(0.3)
    r = live_run(dev, sc, "splitkernel", b, w.options(timeline=False, power_governor=True))
    out[g] = {"exclusive_att": att(ex["requests"]["rows"]), "splitkernel_att": att(r["requests"]["rows"]),
              "n": len(r["requests"]["rows"]), "lp": r["lp"]["tiles_per_s"] / exlp["lp"]["tiles_per_s"],
              "ex_step_p50_us": ex["hp_chain_duration"]["p50_ns"] / 1e3,
              "ex_step_p99_us": ex["hp_chain_duration"]["p99_ns"] / 1e3,
              "sk_step_p50_us": r["hp_chain_duration"]["p50_ns"] / 1e3,
              "sk_step_p99_us": r["hp_chain_duration"]["p99_ns"] / 1e3,
              "ring_p99_us": r["ring_to_first_hp_cta_all"]["p99_ns"] / 1e3}
print(json.dumps(out, indent=1))
dev.close()
