"""Per-CTA phase stamps (live option debug_stamps) of preempted LP runs on configs 2/3:
for each run, the max over CTAs of seen / producer done / MMA done / epilogue done /
teardown / exit begin / last exit (us after the raise), slowest runs first."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200 import live as L  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402

names = ["seen", "prod_done", "mma_done", "epi_done", "teardown", "exit_begin", "last"]
H = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
dev = Device(0)
out = {}
for cls in ("Config3", "Config2"):
    w = getattr(L, cls)(dev)
    w.calibrate()
    sc = w.scenario(seed=11, horizon_s=H, rate=w.hp_rate())
    r = L.live_run(dev, sc, "splitkernel", w.binding(), w.options(timeline=False, power_governor=True, debug_stamps=400))
    runs = r.get("debug_phases", [])
    ks = r.get("debug_kernels", [])
    rows = []
    for k, run in zip(ks, runs):
        mx = {n: (round(run[i][2] / 1e3, 2) if run[i] else None) for i, n in enumerate(names)}
        mn = {n: (round(run[i][0] / 1e3, 2) if run[i] else None) for i, n in enumerate(names)}
        rows.append({"kernel": k, "max": mx, "min_seen": mn["seen"], "late": run[7] if len(run) > 7 else None,
                     "counts": run[8] if len(run) > 8 else None})
    # runs whose first CTA saw the raise > 6 us late were still launching (queued runs, not a drain)
    q = [x for x in rows if x["min_seen"] is not None and x["min_seen"] > 6.0]
    rows = [x for x in rows if x["min_seen"] is not None and x["min_seen"] <= 6.0]
    rows.sort(key=lambda x: -(x["max"]["last"] or 0))
    out[cls] = {"runs": len(rows), "queued_runs": len(q), "exit": r["preempt_flag_to_last_lp_exit"],
                "slowest": rows[:20]}
    w.close()
print(json.dumps(out, indent=1))
dev.close()
