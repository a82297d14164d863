"""Config-4 SLO loss under split-kernel: per request (matched by index on the same trace),
TTFT / TPOT of split-kernel vs exclusive, which SLO bound fails, and the per-token cost
split into ring -> first HP CTA (LP in flight vs idle) and HP step duration."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200 import live as L  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402

H = float(sys.argv[1]) if len(sys.argv) > 1 else 15.0
dev = Device(0)
w = L.Config4(dev)
w.calibrate()
rate = w.hp_rate(0.8)
sc = w.scenario(seed=7, horizon_s=H, rate=rate)
ex = L.live_run(dev, sc, "exclusive", w.binding(), w.options(timeline=False))
sk = L.live_run(dev, sc, "splitkernel", w.binding(), w.options(timeline=False, power_governor=True))
slo = ex["own_p99"]
rx, rs = ex["requests"]["rows"], sk["requests"]["rows"]
n = min(len(rx), len(rs))
fail_ttft = sum(1 for i in range(n) if rs[i][4] and rs[i][1] > slo["ttft_ns"])
fail_tpot = sum(1 for i in range(n) if rs[i][4] and rs[i][2] > slo["tpot_ns"])
d_ttft = sorted((rs[i][1] - rx[i][1]) / 1e3 for i in range(n) if rs[i][4] and rx[i][4])
d_tpot = sorted((rs[i][2] - rx[i][2]) / 1e3 for i in range(n) if rs[i][4] and rx[i][4])


def q(v, f):
    return round(v[min(len(v) - 1, int(f * len(v)))], 2) if v else None


out = {"requests": n, "slo_ns": slo, "ex_fail_ttft": sum(1 for r in rx if r[4] and r[1] > slo["ttft_ns"]),
       "ex_fail_tpot": sum(1 for r in rx if r[4] and r[2] > slo["tpot_ns"]),
       "sk_fail_ttft": fail_ttft, "sk_fail_tpot": fail_tpot,
       "d_ttft_us": {"p10": q(d_ttft, .1), "p50": q(d_ttft, .5), "p90": q(d_ttft, .9)},
       "d_tpot_us": {"p10": q(d_tpot, .1), "p50": q(d_tpot, .5), "p90": q(d_tpot, .9)},
       "ex_step": ex["hp_chain_duration"], "sk_step": sk["hp_chain_duration"],
       "ex_ring": ex["ring_to_first_hp_cta_all"], "sk_ring_inflight": sk["preempt_ring_to_first_hp_cta_lp_in_flight"],
       "sk_ring_idle": sk["preempt_ring_to_first_hp_cta_lp_idle"], "sk_lp_exit": sk["preempt_flag_to_last_lp_exit"],
       "sk_detect_lag": sk["hp_done_detect_lag"], "ex_detect_lag": ex["hp_done_detect_lag"],
       "sk_timer_late": sk["bubble_timer_late"], "ex_timer_late": ex["bubble_timer_late"]}
print(json.dumps(out, indent=1))
dev.close()
