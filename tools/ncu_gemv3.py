"""ncu target: 3 decode layers of the bs=1 GEMV chain (12 ops) — per-PC stall attribution."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device
from paper_2601_04071_b200.live import Config4, decode_step_ops
dev = Device(0)
w = Config4(dev, m=1)
ch = dev.hp_register_chain(decode_step_ops(w.M, w.H, w.Q, w.F, w.V, 16, w.bufs, w.weights, w.lm)[:64])
for i in range(3):
    dev.hp_launch_direct(ch, dev.hp_next_seq())
    dev.sync()
dev.close()
