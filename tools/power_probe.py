"""Development probe: HP SLO / LP throughput / HP chain time / SM clocks of splitkernel with
the LP SM footprint capped inside HP requests (live option small_bubble_sms).
usage: power_probe.py <cfg 1|4> <horizon_s> <sms,...> [extra options json] [option name]
       (0 = no cap; option name defaults to small_bubble_sms, e.g. lp_max_sms)"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import ClockSampler  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, Config4, live_run  # noqa: E402


def pct(d, k):
    return round(d[k] / 1e3, 1) if k in d else None


def main():
    cfg, horizon = sys.argv[1], float(sys.argv[2])
    caps = [int(x) for x in sys.argv[3].split(",")]
    extra = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
    knob = sys.argv[5] if len(sys.argv) > 5 else "small_bubble_sms"
    dev = Device(0)
    w = Config1(dev) if cfg == "1" else Config4(dev)
    w.calibrate()
    sc = w.scenario(seed=7, horizon_s=horizon)
    with ClockSampler(0) as clk:
        ex = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
    slo = {"ttft_ns": ex["own_p99"]["ttft_ns"], "tpot_ns": ex["own_p99"]["tpot_ns"]}
    ex2 = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False, slo=slo))
    exlp = live_run(dev, sc, "exclusive_lp", w.binding(), w.options(timeline=False))
    res = {"exclusive": {"slo": ex2["slo_attainment"], "chain_p50_us": pct(ex["hp_chain_duration"], "p50_ns"),
                         "chain_p90_us": pct(ex["hp_chain_duration"], "p90_ns"), "clocks": clk.summary(),
                         "requests": ex["requests"]["n"]}}
    print("exclusive", json.dumps(res["exclusive"]), flush=True)
    for cap in caps:
        with ClockSampler(0) as clk:
            r = live_run(dev, sc, "splitkernel", w.binding(),
                         w.options(timeline=False, slo=slo, **{knob: cap}, **extra))
        b = {"slo": r["slo_attainment"], "lp_norm": r["lp"]["tiles_per_s"] / max(1e-9, exlp["lp"]["tiles_per_s"]),
             "chain_p50_us": pct(r["hp_chain_duration"], "p50_ns"), "chain_p90_us": pct(r["hp_chain_duration"], "p90_ns"),
             "ring_p99_us": pct(r["preempt_ring_to_first_hp_cta"], "p99_ns"),
             "exit_p50_us": pct(r["preempt_flag_to_last_lp_exit"], "p50_ns"),
             "exit_p90_us": pct(r["preempt_flag_to_last_lp_exit"], "p90_ns"), "clocks": clk.summary(),
             "governor": r.get("power_governor")}
        res[f"split_{knob}{cap}"] = b
        print(f"splitkernel {knob}={cap}", json.dumps(b), flush=True)
    (ROOT / "gpurun_out" / f"power_probe_cfg{cfg}.json").write_text(json.dumps(res, indent=1))
    dev.close()


if __name__ == "__main__":
    main()
