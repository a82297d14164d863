"""Development probe: LP tcgen05 GEMM 8192^3 time (CUDA events, 5 back-to-back full runs,
preemptible) and a non-preemptible timing (host clock over 5 runs); MMA queue lag via
MS_LP_MMA_LAG, single-CTA kernel via MS_LP_GEMM_1SM."""
import ctypes as C
import json
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_04071_b200.live import Config1  # noqa: E402
from paper_2601_04071_b200.device import Device, lib  # noqa: E402
dev = Device(0)
w = Config1(dev)
ms = min(dev.lp_time_full(w.lp, 5) for _ in range(3))
L = lib()
best = 1e9
for _ in range(3):
    dev.sync()
    t = time.perf_counter()
    for _ in range(5):
        L.ms_lp_reset(dev._h, w.lp.id)
        L.ms_lp_run_ex(dev._h, w.lp.id, 0, w.lp.total_tiles, w.lp.total_tiles, 1)
    dev.lp_wait(w.lp, 60)
    dev.sync()
    best = min(best, (time.perf_counter() - t) / 5 * 1e3)
print(json.dumps({"tiles": w.lp.total_tiles, "ms": ms, "tflops": 2 * 8192 ** 3 / (ms * 1e-3) / 1e12,
                  "np_ms": best, "np_tflops": 2 * 8192 ** 3 / (best * 1e-3) / 1e12}), flush=True)
dev.close()
