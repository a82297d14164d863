"""Per-CTA breakdown of an LP GEMM preemption (diagnostics)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2601_04071_b200.device import Device
from paper_2601_04071_b200.live import Config1
dev = Device(0)
w = Config1(dev)
off, _ = dev.calibrate(200)
names = ["seen", "prod_done", "mma_done", "epi_done", "teardown", "exit_begin", "last", "tiles_atom", "exit_atom"]
for trial in range(6):
    dev.lp_reset(w.lp)
    dev.debug_stamps(True)
    dev.lp_run(w.lp, 0, w.lp.total_tiles)
    t = time.perf_counter() + 0.0004
    while time.perf_counter() < t:
        pass
    _, t_raise = dev.preempt_raise()
    st = dev.lp_wait(w.lp, 30)
    dx = np.array(dev.debug_stamps_ext(148), dtype=np.float64)[:, :2]
    d = np.array(dev.debug_stamps(False), dtype=np.float64)
    d = np.concatenate([d[:, :7], dx], axis=1)
    raise_dev = t_raise + off
    rel = (d - raise_dev) / 1e3
    rel[d == 0] = np.nan
    print(f"trial {trial}: exit {(st['t_exit'] - raise_dev)/1e3:.2f}us  seen-first {(st['t_seen']-raise_dev)/1e3:.2f}")
    for i, n in enumerate(names):
        col = rel[:, i]
        col = col[~np.isnan(col)]
        if len(col):
            print(f"   {n:10s} n={len(col):3d} min {col.min():7.2f} p50 {np.median(col):7.2f} max {col.max():7.2f}")
    slow = np.nanargmax(rel[:, 5])
    print("   slowest CTA", slow, [None if np.isnan(x) else round(x, 2) for x in rel[slow]])
dev.close()
