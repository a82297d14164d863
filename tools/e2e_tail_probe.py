"""e2e tail on B200: ring -> HP input resident (SM pull of the 1 MB request input from pinned
host memory, MS_E2E_MODE=2) under split-kernel LP vs an idle GPU, split into ring -> gate
(doorbell seen) and gate -> input resident, p50 / p90 / p99, for pull grids of argv[1:]
CTAs (MS_PULL_CTAS is read once per process, so each size runs in its own process)."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2601_04071_b200.device import Device  # noqa: E402
    from paper_2601_04071_b200.live import Config1, live_run  # noqa: E402

    def pct(xs, q):
        s = sorted(xs)
        return round(s[min(len(s) - 1, int(q * len(s)))] / 1e3, 2) if s else None

    dev = Device(0)
    w = Config1(dev)
    w.calibrate(reps=2, profile=False)
    out = {}
    for pol in ("exclusive", "splitkernel", "exclusive", "splitkernel"):
        r = live_run(dev, w.scenario(seed=77, horizon_s=2.0), pol, w.binding(e2e=True), w.options(timeline=False))
        smp = r["samples"]
        a = smp["ring_to_first_hp_cta_all"]
        o = out.setdefault(pol, {"all": [], "inflight": [], "idle": []})
        o["all"] += a
        o["inflight"] += smp["preempt_ring_to_first_hp_cta_lp_in_flight"]
        o["idle"] += smp["preempt_ring_to_first_hp_cta_lp_idle"]
        o["gate_to_first"] = r["gate_to_first_hp_cta_device"]
    res = {pol: {k: [pct(v, .5), pct(v, .9), pct(v, .99), len(v)] for k, v in o.items() if k != "gate_to_first"}
           | {"gate_to_first_last_run": o["gate_to_first"]} for pol, o in out.items()}
    print(json.dumps(res))
    dev.close()
    sys.exit(0)

res = {}
for n in (sys.argv[1:] or ["7", "14"]):
    env = dict(os.environ, MS_PULL_CTAS=n)
    p = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True, timeout=600)
    res[f"pull_ctas={n}"] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-800:]
print(json.dumps({"how": __doc__.split("\n")[0], "rows": "[p50, p90, p99, n] us", **res}, indent=1))
