"""e2e request-input path on B200: where do the ~48 us of ring ->
first HP CTA go when the HP request's 1 MB input comes from pinned host memory?
  (1) a bare 1 MB pinned H2D copy (host wall, synchronous, 200 reps);
  (2) ring -> first HP CTA of the e2e chain on an idle GPU (exclusive policy) and under LP
      (splitkernel): MS_E2E_MODE=2 SM pull from pinned memory on the HP stream (default;
      first-CTA stamp = input resident), =1 copy engine on its own gated stream + event,
      =0 copy queued behind the HP gate."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, live_run  # noqa: E402


def pct(xs, q):
    s = sorted(xs)
    return s[min(len(s) - 1, int(q * len(s)))] / 1e3 if s else None


dev = Device(0)
w = Config1(dev)
w.calibrate(reps=2)
t = []
for _ in range(200):  # pinned source (the e2e chain's own host buffer)
    t0 = time.perf_counter()
    dev.h2d(w.act[0], w.host_in, w.io_bytes)
    t.append(time.perf_counter() - t0)
out = {"h2d_1MB_sync_us": {"p50": 1e6 * sorted(t)[100], "min": 1e6 * min(t)}}
for mode in ("2", "1", "0"):  # SM pull / copy engine + event / copy behind the gate
    os.environ["MS_E2E_MODE"] = mode
    for pol in ("exclusive", "splitkernel"):
        r = live_run(dev, w.scenario(seed=77, horizon_s=1.0), pol, w.binding(e2e=True), w.options(timeline=False))
        a = r["samples"]["ring_to_first_hp_cta_all"]
        out[f"mode={mode} {pol}"] = {"p50": pct(a, 0.5), "p99": pct(a, 0.99), "n": len(a),
                                        "gate_to_first_p50": r["gate_to_first_hp_cta_device"].get("p50_ns", 0) / 1e3,
                                        "chain_p50": r["hp_chain_duration"].get("p50_ns", 0) / 1e3}
    r = live_run(dev, w.scenario(seed=77, horizon_s=1.0), "exclusive", w.binding(), w.options(timeline=False))
    out[f"no-copy exclusive (ref) {mode}"] = {"p50": pct(r["samples"]["ring_to_first_hp_cta_all"], 0.5)}
print(json.dumps(out, indent=1))
dev.close()
