"""Fused HP chain timeline: alone vs right after preempting the LP GEMM (diagnostics).
Times are us from the doorbell ring (device clock, calibrated)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2601_04071_b200.device import Device
from paper_2601_04071_b200.live import Config1

dev = Device(0)
w = Config1(dev)
off, _ = dev.calibrate(200)
ev = ["p_first_B", "p_A_ready", "p_last_ld", "m_first", "m_commit", "e_tmem", "e_stored", "e_arrived"]


def spin(s):
    t = time.perf_counter() + s
    while time.perf_counter() < t:
        pass


def trial(coloc):
    seq = dev.hp_next_seq()
    dev.debug_stamps(True)  # before arming: the chain's kernel parameters capture the buffer
    dev.hp_arm(w.chain, seq)
    if coloc:
        dev.lp_reset(w.lp)
        dev.lp_run(w.lp, 0, w.lp.total_tiles)
        spin(0.0004)
    else:
        spin(0.0003)
    if coloc:
        _, t_raise = dev.preempt_raise()
    t_ring = dev.hp_ring(seq)
    tm = dev.hp_wait(w.chain, seq, 10)
    st = dev.lp_wait(w.lp, 30) if coloc else None
    d = np.array(dev.debug_stamps_ext(148), dtype=np.float64)
    ring_dev = t_ring + off
    res = {"first": (tm["t_first_cta"] - ring_dev) / 1e3, "done": (tm["t_done"] - ring_dev) / 1e3,
           "gate": (tm["t_gate"] - ring_dev) / 1e3}
    if st:
        res["lp_exit"] = (st["t_exit"] - ring_dev) / 1e3
    for oi in range(4):
        for k in (3, 4, 7):
            x = d[:128, oi * 8 + k]
            x = x[x > 0]
            res[f"op{oi}_{ev[k]}"] = ((np.median(x) - ring_dev) / 1e3, (np.max(x) - ring_dev) / 1e3) if len(x) else None
    return res


for coloc in (False, True):
    rs = [trial(coloc) for _ in range(8)][2:]
    print("=== co-located" if coloc else "=== alone")
    keys = rs[0].keys()
    for k in keys:
        v = [r[k] for r in rs if r[k] is not None]
        if not v:
            continue
        if isinstance(v[0], tuple):
            print(f"  {k:14s} median-CTA {np.median([a for a, b in v]):7.2f}  last-CTA {np.median([b for a, b in v]):7.2f}")
        else:
            print(f"  {k:14s} {np.median(v):7.2f}")
dev.close()
