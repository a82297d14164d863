"""Controlled single-tile GEMM launches for ncu (diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device
dev = Device(0)
a = dev.alloc(128 * 8192 * 2); w = dev.alloc(8192 * 8192 * 2); c = dev.alloc(8192 * 8192 * 2)
dev.fill_synth(a, 128 * 8192, 1, 1, 1.0); dev.fill_synth(w, 8192 * 8192, 1, 2, 1 / 64)
for (n, k) in [(128, 64), (128, 4096), (4096, 4096)]:
    ch = dev.hp_register_chain([dict(kind=1, block_n=128, a=a, b=w, c=c, bias=0, m=128, n=n, k=k, split_k=1, b_layout=1)])
    for _ in range(3):
        dev.hp_launch_direct(ch, dev.hp_next_seq())
        dev.sync()
dev.close()
