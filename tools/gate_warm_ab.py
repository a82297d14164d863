"""Gate L2 warm-up A/B (MS_GATE_WARM_KB, read once per process): live config-1 split-kernel
windows — HP chain duration (first HP CTA -> done), ring -> first HP CTA, request TTFT."""
import json
import os
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, live_run  # noqa: E402

dev = Device(0)
w = Config1(dev)
w.calibrate(2, profile=False)
out = {"warm_kb": os.environ.get("MS_GATE_WARM_KB", "default(2)")}
for pol in ("exclusive", "splitkernel"):
    durs, rings, ttft = [], [], []
    for k in range(3):
        r = live_run(dev, w.scenario(seed=11 + k, horizon_s=2.0), pol, w.binding(), w.options(timeline=False))
        durs.append(r["hp_chain_duration"].get("p50_ns", 0) / 1e3)
        rings += r["samples"]["ring_to_first_hp_cta_all"]
        ttft += [x[1] / 1e3 for x in r["requests"]["rows"] if x[4]]
    rings.sort(); ttft.sort()
    out[pol] = {"chain_p50_us": round(statistics.median(durs), 2),
                "ring_p50_us": round(rings[len(rings) // 2] / 1e3, 2), "ring_p99_us": round(rings[int(0.99 * len(rings))] / 1e3, 2),
                "ttft_p50_us": round(ttft[len(ttft) // 2], 1), "ttft_p90_us": round(ttft[int(0.9 * len(ttft))], 1)}
print(json.dumps(out), flush=True)
dev.close()
