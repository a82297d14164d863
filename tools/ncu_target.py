"""Short, deterministic launch sequence of every tenant kernel for ncu captures
(no live scheduling: ncu serialises and replays kernels)."""
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1  # noqa: E402

dev = Device(0)
w = Config1(dev)
for _ in range(2):                       # LP GEMM 8192^3, full range
    dev.lp_run(w.lp, 0, w.lp.total_tiles)
    dev.lp_wait(w.lp, 60)
for _ in range(2):                       # HP chain: 4 GEMMs + bias/GELU
    dev.hp_launch_direct(w.chain, 0)
    dev.sync()
n = 1 << 30                              # LP HBM streamer, 2^30 bf16
x, y = dev.alloc(2 * n), dev.alloc(2 * n)
dev.fill_synth(x, n, 1, 21, 1.0)
dev.fill_synth(y, n, 1, 22, 1.0)
k = dev.lp_register_axpy(x, y, n, 0.5)
for _ in range(2):
    dev.lp_run(k, 0, k.total_tiles)
    dev.lp_wait(k, 60)
dev.close()
print("ncu target done")
