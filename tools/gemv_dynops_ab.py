"""A/B of the GEMV chain's dynamic prefix (MS_GEMV_DYN_OPS = ops whose units are claimed
dynamically before the static plan takes over) on config 4: the chain alone (best of 3 x 5
steps) and live exclusive vs split-kernel (governed) on the same trace windows, interleaved.
One process per setting (the knob is read once)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(H, seed):
    sys.path.insert(0, ROOT)
    from paper_2601_04071_b200 import live as L
    from paper_2601_04071_b200.device import Device
    dev = Device(0)
    w = L.Config4(dev)
    w.calibrate()
    alone = min(dev.hp_time_chain(w.chain, 5) for _ in range(3))
    rate = w.hp_rate(0.8)
    ex_steps, sk_steps, ring, infl, exr, skr = [], [], [], [], [], []
    for k in range(2):
        sc = w.scenario(seed=seed + 101 * k, horizon_s=H / 2, rate=rate)
        ex = L.live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
        sk = L.live_run(dev, sc, "splitkernel", w.binding(), w.options(timeline=False, power_governor=True))
        ex_steps.append(ex["hp_chain_duration"]["p50_ns"] / 1e3)
        sk_steps.append(sk["hp_chain_duration"]["p50_ns"] / 1e3)
        infl += sk["samples"].get("preempt_ring_to_first_hp_cta_lp_in_flight", [])
        exr += ex["requests"]["rows"]
        skr += sk["requests"]["rows"]
    tt = sorted(r[1] for r in exr if r[4])
    tp = sorted(r[2] for r in exr if r[4])
    slo = (tt[min(len(tt) - 1, int(0.99 * len(tt)))], tp[min(len(tp) - 1, int(0.99 * len(tp)))])
    att = lambda rows: sum(1 for r in rows if r[4] and r[1] <= slo[0] and r[2] <= slo[1]) / max(1, len(rows))  # noqa
    infl.sort()
    print(json.dumps({"alone_ms": round(alone, 4), "ex_step_p50_us": ex_steps, "sk_step_p50_us": sk_steps,
                      "inflight_p50_us": infl[len(infl) // 2] / 1e3 if infl else None,
                      "ex_att": round(att(exr), 4), "sk_att": round(att(skr), 4), "n": len(exr)}), flush=True)
    dev.close()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(float(sys.argv[2]), int(sys.argv[3]))
        sys.exit(0)
    H = float(sys.argv[1]) if len(sys.argv) > 1 else 16.0
    settings = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "2", "4"])]
    for rnd in range(2):
        for n in settings:
            env = dict(os.environ, MS_GEMV_DYN_OPS=str(n))
            r = subprocess.run([sys.executable, __file__, "--one", str(H), str(7 + rnd)], env=env, capture_output=True,
                               text=True, timeout=900)
            line = [x for x in r.stdout.splitlines() if x.startswith("{")]
            row = {"dyn_ops": n, "round": rnd, **(json.loads(line[-1]) if line else {"err": r.stderr[-800:]})}
            print(json.dumps(row), flush=True)
