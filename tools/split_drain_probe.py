"""Where does the drain of a preempted k-split LP GEMM go?  Per CTA (globaltimer, us after
the raise): seen / producer done / MMA done / epilogue done / teardown / exit begin, and the
epilogue's last unit: start (ext 10), TMEM drained + partial stored (11), arrival (12), a
group reduced (13), parked at a chunk boundary (14).  Prints the slowest CTA of each trial."""
import json
import math
import random
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.tenants import block_n_for, split_for  # noqa: E402

dev = Device(0)
off, _ = dev.calibrate(200)
names = ["seen", "prod_done", "mma_done", "epi_done", "teardown", "exit_begin", "last"]
ext = {10: "epi_unit", 11: "stored", 12: "arrived", 13: "reduced", 14: "parked"}
out = {}
random.seed(1)
for (m, n, k) in [(3200, 512, 4608), (128, 192, 802816), (768, 3072, 4096), (12544, 256, 1024)]:
    sp = split_for(m, n, k)
    a, b, c = dev.alloc(m * k * 2), dev.alloc(n * k * 2), dev.alloc(m * n * 2)
    dev.fill_synth(a, m * k, 3, 1, 1.0)
    dev.fill_synth(b, n * k, 3, 2, float(1 / math.sqrt(k)))
    kern = dev.lp_register_gemm(a, b, c, m, n, k, block_n=block_n_for(n), split_k=sp)
    full_ms = dev.lp_time_full(kern, 2)
    rows = []
    for trial in range(8):
        dev.lp_reset(kern)
        dev.debug_stamps(True)
        dev.lp_run(kern, 0, kern.total_tiles)
        t = time.perf_counter() + random.uniform(0.2, 0.9) * full_ms * 1e-3 + 20e-6
        while time.perf_counter() < t:
            pass
        _, t_raise = dev.preempt_raise()
        st = dev.lp_wait(kern, 30)
        dx = np.array(dev.debug_stamps_ext(148), dtype=np.float64)
        d = np.array(dev.debug_stamps(False), dtype=np.float64)
        raise_dev = t_raise + off
        rel = (d[:, :7] - raise_dev) / 1e3
        rel[d[:, :7] == 0] = np.nan
        rx = (dx - raise_dev) / 1e3
        rx[dx == 0] = np.nan
        slow = int(np.nanargmax(rel[:, 5])) if np.any(~np.isnan(rel[:, 5])) else 0
        rows.append({"exit_us": round((st["t_exit"] - raise_dev) / 1e3, 2), "preempted": st["preempted"],
                     "cursor": st["cursor"], "redo": st["redo_count"],
                     "slowest_cta": slow,
                     "phases": {nm: (None if np.isnan(rel[slow, i]) else round(rel[slow, i], 2)) for i, nm in enumerate(names)},
                     "epilogue": {nm: (None if np.isnan(rx[slow, s]) else round(rx[slow, s], 2)) for s, nm in ext.items()},
                     "max_over_ctas": {nm: (None if np.all(np.isnan(rel[:, i])) else round(np.nanmax(rel[:, i]), 2))
                                       for i, nm in enumerate(names)}})
    out[f"{m}x{n}x{k}/split{sp}"] = {"full_ms": round(full_ms, 4), "units": kern.total_tiles, "trials": rows}
    dev.lp_unregister(kern)
    for p_ in (a, b, c):
        dev.free(p_)
print(json.dumps(out, indent=1))
dev.close()
