"""Development probe: HBM streamer (LP axpy, 2^30 bf16) bandwidth and the preemption
it costs an armed HP chain (ring -> first HP CTA, flag -> last LP exit) per
(ctas_per_sm, tile_elems)."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1  # noqa: E402


def spin(s):
    t = time.perf_counter() + s
    while time.perf_counter() < t:
        pass


dev = Device(0)
c1 = Config1(dev)
n = 1 << 30
x, y = dev.alloc(2 * n), dev.alloc(2 * n)
dev.fill_synth(x, n, 1, 21, 1.0)
dev.fill_synth(y, n, 1, 22, 1.0)
for cps, tile in [(4, 8192), (4, 4096), (4, 8192)]:
    k = dev.lp_register_axpy(x, y, n, 0.5, tile_elems=tile, ctas_per_sm=cps)
    ms = dev.lp_time_full(k, 3)
    off, _ = dev.calibrate(100)
    r2f, ex = [], []
    for trial in range(25):
        seq = dev.hp_next_seq()
        dev.hp_arm(c1.chain, seq)
        spin(300e-6)
        dev.lp_reset(k)
        dev.lp_run(k, 0, k.total_tiles)
        spin(300e-6)
        _, t_raise = dev.preempt_raise()
        t_ring = dev.hp_ring(seq)
        t = dev.hp_wait(c1.chain, seq, 10)
        st = dev.lp_wait(k, 30)
        r2f.append((t["t_first_cta"] - off - t_ring) / 1e3)
        if st["preempted"]:
            ex.append((st["t_exit"] - off - t_raise) / 1e3)
        dev.sync()
    print(f"ctas/SM {cps} tile {tile:6d}: {6 * n / (ms * 1e-3) / 1e12:.2f} TB/s | ring->first HP CTA p50 "
          f"{np.percentile(r2f, 50):.2f} p90 {np.percentile(r2f, 90):.2f} | flag->last LP exit p50 "
          f"{np.percentile(ex, 50) if ex else float('nan'):.2f} p90 {np.percentile(ex, 90) if ex else float('nan'):.2f}", flush=True)
    dev.lp_unregister(k)
dev.close()
