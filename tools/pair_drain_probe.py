"""Where the CTA-pair LP GEMM drain goes (standalone, no HP): the 8192^3 pair GEMM is
launched, preempted 150-550 us in, and every CTA's phase stamps (tile_run.cuh / tc_gemm2.cuh
dbg slots) are read back, relative to the host raise (clock offset from ms_clock_calibrate).
Per phase: p50 / p90 over runs of the max over CTAs (and of the min), plus the CTAs most
often last.  argv[1]: runs (default 40)."""
import collections
import ctypes as C
import json
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device, lib  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 40
n = 8192
dev = Device(0)
a, b, c = dev.alloc(n * n * 2), dev.alloc(n * n * 2), dev.alloc(n * n * 2)
dev.fill_synth(a, n * n, 1, 1, 1.0)
dev.fill_synth(b, n * n, 1, 2, 1.0 / 90.5)
k = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
off, rtt = dev.calibrate()
base = {0: "seen", 1: "prod_done", 2: "mma_done", 3: "epi_done", 4: "teardown", 5: "exit_begin", 6: "exit_record"}
ext = {1: "cta0_count_complete", 20: "lead_prod_stop", 21: "peer_report_rcvd", 22: "terminal_issued",
       23: "peer_prod_stop", 24: "mma_saw_preempt", 25: "mma_positions_consumed", 26: "mma_drained",
       27: "mma_abort_signalled", 28: "epi_abort_seen", 29: "epi_end_seen", 30: "host_poller_left",
       31: "mirror_poller_left"}
NW = 2048 + 148 * 64
per = collections.defaultdict(lambda: {"max": [], "min": [], "argmax": collections.Counter()})
drains, frees = [], []
rng = random.Random(5)
for r in range(runs):
    dev.lp_reset(k)
    dev.debug_stamps(True)
    dev.lp_run(k, 0, k.total_tiles)
    t_end = time.perf_counter() + rng.uniform(150e-6, 550e-6)
    while time.perf_counter() < t_end:
        pass
    _, t_host = dev.preempt_raise()
    st = dev.lp_wait(k, 30)
    buf = (C.c_ulonglong * NW)()
    lib().ms_debug_stamps(dev._h, 0, buf, NW)
    if not st["preempted"]:
        continue
    t0 = t_host + off
    drains.append((st["t_exit"] - t0) / 1e3)
    frees.append((st["t_free"] - t0) / 1e3)
    for ph, name in list(base.items()) + [(100 + e, v) for e, v in ext.items()]:
        vals = []
        for cta in range(148):
            v = buf[cta * 8 + ph] if ph < 100 else buf[2048 + cta * 64 + (ph - 100)]
            if v:
                vals.append(((v - t0) / 1e3, cta))
        if vals:
            mx = max(vals)
            per[name]["max"].append(mx[0])
            per[name]["min"].append(min(vals)[0])
            per[name]["argmax"][mx[1]] += 1


def q(v, f):
    v = sorted(v)
    return round(v[min(len(v) - 1, int(f * len(v)))], 2) if v else None


out = {"runs_preempted": len(drains), "clock_rtt_ns": rtt,
       "flag_to_exit_record_us": [q(drains, .5), q(drains, .9), q(drains, .99)],
       "flag_to_sms_free_us": [q(frees, .5), q(frees, .9), q(frees, .99)], "phases_us": {}}
for name, d in per.items():
    out["phases_us"][name] = {"max_p50": q(d["max"], .5), "max_p90": q(d["max"], .9), "min_p50": q(d["min"], .5),
                              "n": len(d["max"]), "last_ctas": d["argmax"].most_common(3)}
print(json.dumps(out, indent=1))
dev.close()
