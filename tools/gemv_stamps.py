"""Per-op timeline of the bs=1 GEMV chain (SM-cycle debug stamps, hp_gemv.cuh gemv_stamp):
3 decode layers (12 ops).  Per op, median/max over CTAs of the time since the CTA's start
(us at the SM clock ncu reports): input phase passed, x in smem, consumer done, arrived,
and the producer's last-unit issue."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2601_04071_b200.device import Device
from paper_2601_04071_b200.live import Config4, decode_step_ops
GHZ = float(sys.argv[1]) if len(sys.argv) > 1 else 1.92
dev = Device(0)
w = Config4(dev, m=1)
ops = decode_step_ops(w.M, w.H, w.Q, w.F, w.V, 3, w.bufs, w.weights, w.lm)[:12]
ch = dev.hp_register_chain(ops)
names = ["qkv", "o", "gu", "down"] * 3
G = 147
for trial in range(3):
    dev.sync()
    dev.debug_stamps(True)
    dev.hp_launch_direct(ch, dev.hp_next_seq())
    dev.sync()
    d = np.array(dev.debug_stamps_ext(148), dtype=np.float64)[:G]
    rel = (d - d[:, 63:64]) / (GHZ * 1e3)
    f = lambda x: f"{np.median(x):6.2f}/{np.max(x):6.2f}"
    print(f"--- trial {trial} (us since CTA start, median/max over CTAs)")
    for oi in range(12):
        cols = [f"{nm}={f(rel[:, 4 * oi + k])}" for k, nm in enumerate(["in", "x", "done", "arr"])]
        cols.append(f"prod_last={f(rel[:, 48 + oi])}")
        print(f"op{oi:2d} {names[oi]:5s} " + " ".join(cols))
    import ctypes as C
    from paper_2601_04071_b200.device import lib
dev.sync()
dev.debug_stamps(True)
dev.hp_launch_direct(ch, dev.hp_next_seq())
dev.sync()
import ctypes as C
from paper_2601_04071_b200.device import lib
buf = (C.c_ulonglong * 32768)()
lib().ms_debug_stamps(dev._h, 0, buf, 32768)
a = np.array(buf, dtype=np.float64)
gt = a[2048 + 148 * 64:2048 + 148 * 64 + 148 * 16].reshape(148, 16)[:G]
t0 = gt[gt > 0].min()
print("global time (us): op done [min/med/max over CTAs] -> next op x ready [min/med/max]")
for oi in range(0, 8):
    dn = (gt[:, 8 + oi] - t0) / 1e3
    xr = (gt[:, oi + 1] - t0) / 1e3
    print(f"op{oi}->{oi + 1}: done {dn.min():6.2f}/{np.median(dn):6.2f}/{dn.max():6.2f}  x {xr.min():6.2f}/{np.median(xr):6.2f}/{xr.max():6.2f}"
          f"  slowest-done CTA {int(np.argmax(dn))}")
dev.close()

