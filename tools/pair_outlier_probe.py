"""Hunt rare long preemptions with the CTA-pair LP GEMM (config 1, live): several windows,
report the HP activations with ring -> first HP CTA > 50 us and every preempted LP run
whose flag -> exit or flag -> seen exceeds 50 us (kernel, start / seen / exit vs raise)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, live_run  # noqa: E402

dev = Device(0)
w = Config1(dev)
w.calibrate(reps=2)
out = []
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    r = live_run(dev, w.scenario(seed=21 + k, horizon_s=1.5), "splitkernel", w.binding(), w.options(timeline=False))
    inf = sorted(r["samples"]["preempt_ring_to_first_hp_cta_lp_in_flight"])
    runs = [x for x in r["samples"]["preempted_lp_runs"] if x[1] > 50_000 or (x[3] and x[3] > 50_000)]
    out.append({"window": k, "inflight_n": len(inf), "inflight_top": [round(x / 1e3, 1) for x in inf[-5:]],
                "lp_exit": r["preempt_flag_to_last_lp_exit"], "slow_lp_runs": [[a, b / 1e3, c / 1e3, d / 1e3, e] for a, b, c, d, e in runs]})
    print(json.dumps(out[-1]), flush=True)
dev.close()
