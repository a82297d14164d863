"""Live config-1 A/B of an env knob read by the device layer (one process per setting, two
alternating rounds of two 2.5 s split-kernel windows each, seeds 31/32): ring -> first HP CTA
(all / LP in flight), LP drain (exit record / SMs free), HP request TTFT / TPOT p99, LP GEMM
passes per second, and the LP GEMM's best-of-10 whole-launch TFLOP/s.
Usage: live_env_ab.py VAR v1 v2 ..."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import time
    from paper_2601_04071_b200.device import Device  # noqa: E402
    from paper_2601_04071_b200.live import Config1, live_run  # noqa: E402

    dev = Device(0)
    w = Config1(dev)
    w.calibrate(reps=2, profile=False)
    best = 1e9
    for _ in range(10):
        time.sleep(0.03)
        best = min(best, dev.lp_time_full(w.lp, 1))
    acc = {"all": [], "inflight": [], "lp_exit": [], "lp_free": [], "ttft": [], "tpot": [], "passes": 0.0, "secs": 0.0,
           "tflops": 2 * 8192 ** 3 / (best * 1e-3) / 1e12, "units": w.lp.total_tiles}
    for i in range(2):
        r = live_run(dev, w.scenario(seed=31 + i, horizon_s=2.5), "splitkernel", w.binding(), w.options(timeline=False))
        s = r["samples"]
        acc["all"] += s["preempt_ring_to_first_hp_cta"]
        acc["inflight"] += s["preempt_ring_to_first_hp_cta_lp_in_flight"]
        acc["lp_exit"] += s["preempt_flag_to_last_lp_exit"]
        acc["lp_free"] += s.get("preempt_flag_to_lp_sms_free", [])
        acc["ttft"] += [x[1] for x in r["requests"]["rows"] if x[4]]
        acc["tpot"] += [x[2] for x in r["requests"]["rows"] if x[4]]
        acc["passes"] += r["lp"]["tiles_done"] / w.lp.total_tiles
        acc["secs"] += 2.5
    print(json.dumps(acc))
    dev.close()
    sys.exit(0)


def pct(xs, q):
    s = sorted(xs)
    return round(s[min(len(s) - 1, int(q * len(s)))] / 1e3, 2) if s else None


var, vals = sys.argv[1], sys.argv[2:]
pooled = {}
for rnd in range(2):
    for v in vals:
        env = dict(os.environ, **{var: v})
        p = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True, timeout=900)
        if p.returncode != 0:
            pooled[f"{var}={v}"] = p.stderr[-600:]
            continue
        d = json.loads(p.stdout.strip().splitlines()[-1])
        t = pooled.setdefault(f"{var}={v}", {"lists": {}, "passes": 0.0, "secs": 0.0, "tflops": [], "units": d["units"]})
        for k in ("all", "inflight", "lp_exit", "lp_free", "ttft", "tpot"):
            t["lists"].setdefault(k, []).extend(d[k])
        t["passes"] += d["passes"]
        t["secs"] += d["secs"]
        t["tflops"].append(round(d["tflops"], 1))
out = {}
for k, t in pooled.items():
    if isinstance(t, str):
        out[k] = t
        continue
    o = {kk: [pct(v, .5), pct(v, .99), len(v)] for kk, v in t["lists"].items()}
    o["lp_passes_per_s"] = round(t["passes"] / t["secs"], 2)
    o["tflops_best_of_10"] = t["tflops"]
    o["units_per_pass"] = t["units"]
    out[k] = o
print(json.dumps({"how": __doc__.split("\n")[0], "rows": "[p50, p99, n] us", **out}, indent=1))
