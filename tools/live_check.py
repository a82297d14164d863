"""Development driver: live config-1 runs of every policy on one B200 (prints summaries)."""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, live_run  # noqa: E402


def brief(r: dict) -> dict:
    keys = ["policy", "slo_attainment", "own_p99", "preempt_ring_to_first_hp_cta", "preempt_flag_to_last_lp_exit",
            "ring_to_first_hp_cta_all", "gate_to_first_hp_cta_device", "hp_chain_duration", "lp", "loops"]
    out = {k: r.get(k) for k in keys}
    out["requests"] = {k: v for k, v in r["requests"].items() if k != "rows"}
    return out


def main():
    horizon = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
    dev = Device(0)
    w = Config1(dev)
    calib = w.calibrate()
    print("calib", calib, flush=True)
    sc = w.scenario(seed=1, horizon_s=horizon)
    res = {"calib": calib}
    t = time.time()
    ex = live_run(dev, sc, "exclusive", w.binding(), w.options())
    print("exclusive", json.dumps(brief(ex)), f"{time.time() - t:.1f}s", flush=True)
    slo = {"ttft_ns": ex["own_p99"]["ttft_ns"], "tpot_ns": ex["own_p99"]["tpot_ns"]}
    res["exclusive"] = brief(ex)
    ex2 = live_run(dev, sc, "exclusive", w.binding(), w.options(slo=slo))
    res["exclusive_att"] = ex2.get("slo_attainment")
    print("exclusive attainment vs own slo", res["exclusive_att"], flush=True)
    exlp = live_run(dev, sc, "exclusive_lp", w.binding(), w.options())
    print("exclusive_lp", json.dumps(brief(exlp)), flush=True)
    res["exclusive_lp"] = brief(exlp)
    for pol, kw in [("splitkernel", {}), ("splitkernel", {"eager": True}), ("reef", {}), ("reef_req", {})]:
        t = time.time()
        r = live_run(dev, sc, pol, w.binding(), w.options(slo=slo, **kw,
                     ndjson_path=str(ROOT / "gpurun_out" / f"live_{pol}{'_eager' if kw else ''}.ndjson")))
        b = brief(r)
        b["lp_norm"] = r["lp"]["tiles_per_s"] / max(1e-9, exlp["lp"]["tiles_per_s"])
        print(pol, kw, json.dumps(b), f"{time.time() - t:.1f}s", flush=True)
        res[pol + ("_eager" if kw else "")] = b
    (ROOT / "gpurun_out" / "live_check.json").write_text(json.dumps(res, indent=1))
    dev.close()


if __name__ == "__main__":
    main()
