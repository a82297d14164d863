"""Probe (env MS_LP_CLUSTER_ALIGN / MS_GATE_SMEM set by the caller): LP GEMM throughput and
the preemption an armed config-1 fused chain (4-CTA clusters) / config-4 GEMV chain sees
while the LP GEMM runs: ring -> gate, gate -> first HP CTA, flag -> last LP exit (us)."""
import json
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, Config4  # noqa: E402


def spin(s):
    t = time.perf_counter() + s
    while time.perf_counter() < t:
        pass


dev = Device(0)
c1, c4 = Config1(dev), Config4(dev)
k = c1.lp
ms = min(dev.lp_time_full(k, 3) for _ in range(2))
row = {"align": os.environ.get("MS_LP_CLUSTER_ALIGN", "0"), "gate_smem": os.environ.get("MS_GATE_SMEM", "40960"),
       "lp_gemm_tflops": 2 * 8192 ** 3 / (ms * 1e-3) / 1e12}
for cname, ch in {"cfg1_fused": c1.chain, "cfg4_gemv": c4.chain}.items():
    off, _ = dev.calibrate(100)
    r2g, g2f, ex = [], [], []
    for trial in range(40):
        seq = dev.hp_next_seq()
        dev.hp_arm(ch, seq)
        spin(300e-6)
        dev.lp_reset(k)
        dev.lp_run(k, 0, k.total_tiles)
        spin(300e-6)
        _, t_raise = dev.preempt_raise()
        t_ring = dev.hp_ring(seq)
        t = dev.hp_wait(ch, seq, 10)
        st = dev.lp_wait(k, 30)
        if t["t_gate"]:
            r2g.append((t["t_gate"] - off - t_ring) / 1e3)
            g2f.append((t["t_first_cta"] - t["t_gate"]) / 1e3)
        if st["preempted"]:
            ex.append((st["t_exit"] - off - t_raise) / 1e3)
        dev.sync()
    q = lambda v, p: round(float(np.percentile(v, p)), 2) if v else None  # noqa: E731
    row[cname] = {"ring_gate": [q(r2g, 50), q(r2g, 90)], "gate_first": [q(g2f, 50), q(g2f, 90), q(g2f, 99)],
                  "exit": [q(ex, 50), q(ex, 90)]}
print(json.dumps(row), flush=True)
dev.close()
