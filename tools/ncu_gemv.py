"""ncu target: the bs=1 GEMV decode chain (hp_gemv.cuh) — LM head alone, then the full
config-4 step (argv[1] = 'lm' | 'step' | 'both')."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device
from paper_2601_04071_b200.live import Config4, decode_step_ops
dev = Device(0)
w = Config4(dev, m=1)
ops = decode_step_ops(w.M, w.H, w.Q, w.F, w.V, w.LAYERS, w.bufs, w.weights, w.lm)
what = sys.argv[1] if len(sys.argv) > 1 else "both"
chains = []
if what in ("lm", "both"):
    chains.append(dev.hp_register_chain(ops[-1:]))
if what in ("step", "both"):
    chains.append(w.chain)
for ch in chains:
    for i in range(2):
        dev.hp_launch_direct(ch, dev.hp_next_seq())
        dev.sync()
dev.close()
