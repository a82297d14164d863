"""Development driver: live config-4 runs (decode HP + GEMM and streamer LP) on one B200."""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4, live_run  # noqa: E402
from tools.live_check import brief  # noqa: E402


def main():
    horizon = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
    dev = Device(0)
    w = Config4(dev)
    calib = w.calibrate()
    print("calib", calib, flush=True)
    sc = w.scenario(seed=1, horizon_s=horizon)
    res = {"calib": calib}
    ex = live_run(dev, sc, "exclusive", w.binding(), w.options())
    res["exclusive"] = brief(ex)
    print("exclusive", json.dumps(res["exclusive"]), flush=True)
    slo = {"ttft_ns": ex["own_p99"]["ttft_ns"], "tpot_ns": ex["own_p99"]["tpot_ns"]}
    ex2 = live_run(dev, sc, "exclusive", w.binding(), w.options(slo=slo))
    res["exclusive_att"] = ex2.get("slo_attainment")
    print("exclusive attainment vs own slo", res["exclusive_att"], "rate", sc["traces"][0]["bursty"]["rate"], flush=True)
    exlp = live_run(dev, sc, "exclusive_lp", w.binding(), w.options())
    res["exclusive_lp"] = brief(exlp)
    for pol, kw in [("splitkernel", {}), ("splitkernel", {"eager": True}), ("reef", {}), ("reef_req", {})]:
        r = live_run(dev, sc, pol, w.binding(), w.options(slo=slo, **kw))
        b = brief(r)
        b["lp_norm"] = r["lp"]["tiles_per_s"] / max(1e-9, exlp["lp"]["tiles_per_s"])
        print(pol, kw, json.dumps(b), flush=True)
        res[pol + ("_eager" if kw else "")] = b
    (ROOT / "gpurun_out" / "live_check4.json").write_text(json.dumps(res, indent=1))
    dev.close()


if __name__ == "__main__":
    main()
