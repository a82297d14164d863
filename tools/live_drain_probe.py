"""Where the LP drain goes in LIVE config-1 runs (flag raise -> last LP CTA exit): per-CTA
phase stamps of up to 60 preempted runs (live option debug_stamps), reduced to the
per-run max over CTAs of each phase, then p50 / p90 / max over runs (us after the raise).
Phases (tile_run.cuh / tc_gemm.cuh): seen (CTA observed the epoch), prod_done (TMA
producer stopped), mma_done (queued k-blocks drained), epi_done, teardown, exit_begin,
last (the last CTA's exit record)."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, live_run  # noqa: E402

names = ["seen", "prod_done", "mma_done", "epi_done", "teardown", "exit_begin", "last"]
dev = Device(0)
w = Config1(dev)
w.calibrate(2)
out = {}
for label, extra in (("ungoverned", {}), ("governed", {"power_governor": True})):
    r = live_run(dev, w.scenario(seed=3, horizon_s=2.0), "splitkernel", w.binding(),
                 w.options(timeline=False, debug_stamps=60, **extra))
    runs = r.get("debug_phases", [])
    per = {n: sorted(run[i][2] for run in runs if run[i]) for i, n in enumerate(names)}
    first = {n: sorted(run[i][0] for run in runs if run[i]) for i, n in enumerate(names)}

    def q(v, f):
        return round(v[min(len(v) - 1, int(f * len(v)))] / 1e3, 2) if v else None
    out[label] = {"runs": len(runs), "flag_to_last_exit": r["preempt_flag_to_last_lp_exit"],
                  "max_over_ctas_us": {n: [q(per[n], .5), q(per[n], .9), q(per[n], 1.0)] for n in names},
                  "min_over_ctas_us": {n: [q(first[n], .5), q(first[n], .9)] for n in names}}
print(json.dumps(out, indent=1))
dev.close()
