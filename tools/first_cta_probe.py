"""Development probe: doorbell ring -> gate -> first HP CTA of an armed chain while an LP
kernel occupies the GPU (no scheduler: ring + raise by hand).  Chains: config-1 fused
tcgen05 chain (4-CTA clusters) and config-4 bs=1 GEMV chain; LP: none / GEMM / axpy;
LP SM reserve 1 / 4.  Prints p50/p90 of ring->gate and gate->first (us)."""
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
c1 = Config1(dev)
c4 = Config4(dev)
lps = {"none": None, "gemm": c1.lp, "axpy": c4.lp_axpy}
chains = {"cfg1_fused": c1.chain, "cfg4_gemv": c4.chain}
for reserve in (1, 4):
    dev.set_lp_sm_reserve(reserve)
    for cname, ch in chains.items():
        for lname, lp in lps.items():
            off, _ = dev.calibrate(100)
            r2g, g2f = [], []
            for trial in range(25):
                seq = dev.hp_next_seq()
                dev.hp_arm(ch, seq)
                spin(300e-6)  # the armed chain reaches the GPU (launch latency is not measured)
                if lp is not None:
                    dev.lp_reset(lp)
                    dev.lp_run(lp, 0, lp.total_tiles)
                    spin(300e-6)
                    dev.preempt_raise()
                t_ring = dev.hp_ring(seq)
                t = dev.hp_wait(ch, seq, 10)
                if lp is not None:
                    dev.lp_wait(lp, 30)
                if t["t_gate"]:
                    r2g.append((t["t_gate"] - off - t_ring) / 1e3)
                    g2f.append((t["t_first_cta"] - t["t_gate"]) / 1e3)
                dev.sync()
            q = lambda v, p: float(np.percentile(v, p)) if v else float("nan")  # noqa: E731
            print(f"reserve={reserve} {cname:10s} lp={lname:5s} ring->gate p50 {q(r2g, 50):5.2f} p90 {q(r2g, 90):5.2f}"
                  f" | gate->first p50 {q(g2f, 50):5.2f} p90 {q(g2f, 90):5.2f}", flush=True)
dev.set_lp_sm_reserve(1)
dev.close()
