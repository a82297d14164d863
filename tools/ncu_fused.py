"""ncu target: the fused config-1 HP chain kernel (4 x [128x4096]x[4096x4096]^T + bias/GELU)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device
dev = Device(0)
M, H = 128, 4096
act = [dev.alloc(M * H * 2) for _ in range(5)]
ws = [dev.alloc(H * H * 2) for _ in range(4)]
bias = dev.alloc(H * 2)
dev.fill_synth(act[0], M * H, 1, 100, 1.0)
for i, w in enumerate(ws):
    dev.fill_synth(w, H * H, 1, 101 + i, 1.0 / 64)
dev.fill_synth(bias, H, 1, 110, 0.1)
ops = [dict(kind=1, block_n=128, a=act[i], b=ws[i], c=act[i + 1], bias=0, m=M, n=H, k=H) for i in range(4)]
ops.append(dict(kind=2, block_n=0, a=act[4], b=0, c=act[0], bias=bias, m=M, n=H, k=0))
ch = dev.hp_register_chain(ops)
dev.hp_set_fused(len(sys.argv) < 2 or sys.argv[1] != "perop")
for i in range(3):
    dev.hp_launch_direct(ch, dev.hp_next_seq())
    dev.sync()
dev.close()
