"""A/B of the GEMV chain's head prefetch (MS_GEMV_HEAD_KB) on the config-4 live leg: per
setting (separate process: the knob is read once), exclusive + split-kernel (governed) on
the same trace at 80% HP load; reports SLO attainment, LP, step p50 and ring p99."""
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
    rate = w.hp_rate(0.8)
    sc = w.scenario(seed=seed, horizon_s=H, rate=rate)
    ex = L.live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
    slo = ex["own_p99"]
    att = lambda rows: sum(1 for x in rows if x[4] and x[1] <= slo["ttft_ns"] and x[2] <= slo["tpot_ns"]) / max(1, len(rows))  # noqa
    exlp = L.live_run(dev, w.scenario(seed=seed, horizon_s=3.0, rate=rate), "exclusive_lp", w.binding(),
                      w.options(timeline=False, power_governor=True))
    sk = L.live_run(dev, sc, "splitkernel", w.binding(), w.options(timeline=False, power_governor=True))
    res = {"n": len(ex["requests"]["rows"]), "ex_att": att(ex["requests"]["rows"]), "sk_att": att(sk["requests"]["rows"]),
           "lp": sk["lp"]["tiles_per_s"] / exlp["lp"]["tiles_per_s"],
           "ex_step_p50_us": ex["hp_chain_duration"]["p50_ns"] / 1e3, "sk_step_p50_us": sk["hp_chain_duration"]["p50_ns"] / 1e3,
           "ex_step_p99_us": ex["hp_chain_duration"]["p99_ns"] / 1e3, "sk_step_p99_us": sk["hp_chain_duration"]["p99_ns"] / 1e3,
           "ring_p99_us": sk["ring_to_first_hp_cta_all"]["p99_ns"] / 1e3,
           "inflight_p50_us": sk["preempt_ring_to_first_hp_cta_lp_in_flight"].get("p50_ns", 0) / 1e3}
    print(json.dumps(res), flush=True)
    dev.close()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(float(sys.argv[2]), int(sys.argv[3]))
        sys.exit(0)
    H = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
    settings = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "49152"])]
    out = []
    for rnd in range(2):
        for kb in settings:
            env = dict(os.environ, MS_GEMV_HEAD_KB=str(kb))
            r = subprocess.run([sys.executable, __file__, "--one", str(H), str(7 + rnd)], env=env, capture_output=True,
                               text=True, timeout=900)
            line = [x for x in r.stdout.splitlines() if x.startswith("{")]
            row = {"head_kb": kb, "round": rnd, **(json.loads(line[-1]) if line else {"err": r.stderr[-500:]})}
            out.append(row)
            print(json.dumps(row), flush=True)
