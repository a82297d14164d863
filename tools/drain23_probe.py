"""Which preempted LP runs drain slowly on configs 2/3?  Runs split-kernel (governed) for H s
and prints the slowest preempted runs (kernel, flag -> exit, start/seen vs the raise) and
per-kernel p50/p99 of flag -> last exit."""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200 import live as L  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402

H = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
dev = Device(0)
out = {}
for cls in ("Config2", "Config3"):
    w = getattr(L, cls)(dev)
    w.calibrate()
    sc = w.scenario(seed=11, horizon_s=H, rate=w.hp_rate())
    r = L.live_run(dev, sc, "splitkernel", w.binding(), w.options(timeline=False, power_governor=True))
    allruns = r["samples"]["preempted_lp_runs"]
    runs = [x for x in allruns if x[2] <= 0]  # started before the raise (drain of running LP work)
    runs.sort(key=lambda x: -x[1])
    q = sorted(x[1] for x in runs)
    pct = (lambda f: q[max(0, -(-int(f * len(q)) // 1) - 1)] / 1e3 if q else None)
    per = defaultdict(list)
    for k, ex, st, se, det in runs:
        per[k].append(ex)
    stats = {k: {"n": len(v), "p50_us": sorted(v)[len(v) // 2] / 1e3, "max_us": max(v) / 1e3} for k, v in per.items()}
    out[cls] = {"n": len(runs), "queued": len(allruns) - len(runs), "exit_p50_us": pct(0.5), "exit_p99_us": pct(0.99),
                "lp_exit_summary": r["preempt_flag_to_last_lp_exit"], "slowest": [[k, ex / 1e3, st / 1e3, se / 1e3, det] for k, ex, st, se, det in runs[:25]],
                "per_kernel": dict(sorted(stats.items(), key=lambda kv: -kv[1]["max_us"])[:20])}
    w.close()
print(json.dumps(out, indent=1))
dev.close()
