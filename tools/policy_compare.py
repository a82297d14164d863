"""Development driver: live policy comparison on one B200 for config 1 or 4, optionally
with the power governor on every policy that runs LP work.
usage: policy_compare.py <cfg 1|4> <horizon_s> [governor 0|1] [seed] [config-4 HP utilisation]
                         [extra splitkernel options json]"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import ClockSampler  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, Config4, live_run  # noqa: E402


def main():
    cfg, horizon = sys.argv[1], float(sys.argv[2])
    gov = len(sys.argv) > 3 and sys.argv[3] == "1"
    seed = int(sys.argv[4]) if len(sys.argv) > 4 else 7
    dev = Device(0)
    w = Config1(dev) if cfg == "1" else Config4(dev)
    w.calibrate()
    util = float(sys.argv[5]) if len(sys.argv) > 5 else None
    sc = w.scenario(seed=seed, horizon_s=horizon, rate=w.hp_rate(util)) if (cfg == "4" and util) else \
        w.scenario(seed=seed, horizon_s=horizon)
    ex = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
    slo = {"ttft_ns": ex["own_p99"]["ttft_ns"], "tpot_ns": ex["own_p99"]["tpot_ns"]}
    ex2 = live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False, slo=slo))
    extra = {"power_governor": True} if gov else {}
    sk_extra = json.loads(sys.argv[6]) if len(sys.argv) > 6 else {}
    exlp = live_run(dev, sc, "exclusive_lp", w.binding(), w.options(timeline=False, **extra))
    res = {"config": cfg, "horizon_s": horizon, "governor": gov, "seed": seed, "hp_utilisation": util,
           "rate": sc["traces"][0]["bursty"]["rate"],
           "requests": ex["requests"]["n"], "exclusive_slo": ex2["slo_attainment"],
           "exclusive_lp_tiles_per_s": exlp["lp"]["tiles_per_s"]}
    print("exclusive", res, flush=True)
    for pol in (("splitkernel",) if sk_extra else ("splitkernel", "reef_req", "reef")):
        with ClockSampler(0) as clk:
            r = live_run(dev, sc, pol, w.binding(),
                         w.options(timeline=False, slo=slo, **extra, **(sk_extra if pol == "splitkernel" else {})))
        b = {"slo": r["slo_attainment"], "lp_norm": r["lp"]["tiles_per_s"] / max(1e-9, exlp["lp"]["tiles_per_s"]),
             "ring_p99_us": r["ring_to_first_hp_cta_all"].get("p99_ns", 0) / 1e3,
             "chain_p50_us": r["hp_chain_duration"].get("p50_ns", 0) / 1e3, "clocks": clk.summary(),
             "mean_lp_sms": (r.get("power_governor") or {}).get("mean_lp_sms")}
        res[pol] = b
        print(pol, json.dumps(b), flush=True)
    if "reef_req" in res:
        res["lp_split_over_reef_req"] = res["splitkernel"]["lp_norm"] / max(1e-9, res["reef_req"]["lp_norm"])
        print("lp splitkernel / reef_req =", res["lp_split_over_reef_req"], flush=True)
    (ROOT / "gpurun_out" / f"policy_compare_cfg{cfg}_gov{int(gov)}_u{util or 0.5}.json").write_text(json.dumps(res, indent=1))
    dev.close()


if __name__ == "__main__":
    main()
