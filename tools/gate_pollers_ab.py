"""Doorbell gate pollers A/B on B200: live config-1 split-kernel windows with the HP gate's
doorbell polled by argv[1:] warps (MS_GATE_WARPS, read once per process, so each setting
runs in its own process; settings alternate over two rounds).  Reports ring -> first HP
CTA [p50, p90, p99, n] for all activations, LP-in-flight and LP-idle ones, and the LP drain."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2601_04071_b200.device import Device  # noqa: E402
    from paper_2601_04071_b200.live import Config1, live_run  # noqa: E402

    dev = Device(0)
    w = Config1(dev)
    w.calibrate(reps=2, profile=False)
    acc = {"all": [], "inflight": [], "idle": [], "lp_exit": [], "lp_free": []}
    for i in range(2):
        r = live_run(dev, w.scenario(seed=31 + i, horizon_s=2.5), "splitkernel", w.binding(), w.options(timeline=False))
        s = r["samples"]
        acc["all"] += s["preempt_ring_to_first_hp_cta"]
        acc["inflight"] += s["preempt_ring_to_first_hp_cta_lp_in_flight"]
        acc["idle"] += s["preempt_ring_to_first_hp_cta_lp_idle"]
        acc["lp_exit"] += s["preempt_flag_to_last_lp_exit"]
        acc["lp_free"] += s.get("preempt_flag_to_lp_sms_free", [])
    print(json.dumps(acc))
    dev.close()
    sys.exit(0)


def pct(xs, q):
    s = sorted(xs)
    return round(s[min(len(s) - 1, int(q * len(s)))] / 1e3, 2) if s else None


pooled = {}
for rnd in range(2):
    for n in (sys.argv[1:] or ["4", "16"]):
        env = dict(os.environ, MS_GATE_WARPS=n)
        p = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True, timeout=900)
        if p.returncode != 0:
            pooled[f"gate_warps={n}"] = p.stderr[-600:]
            continue
        d = json.loads(p.stdout.strip().splitlines()[-1])
        tgt = pooled.setdefault(f"gate_warps={n}", {k: [] for k in d})
        for k, v in d.items():
            tgt[k] += v
out = {k: ({kk: [pct(v, .5), pct(v, .9), pct(v, .99), len(v)] for kk, v in d.items()} if isinstance(d, dict) else d)
       for k, d in pooled.items()}
print(json.dumps({"how": __doc__.split("\n")[0], "rows": "[p50, p90, p99, n] us", **out}, indent=1))
