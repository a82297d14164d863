"""Time HP GEMM variants in isolation (128 x 4096 x 4096)."""
import math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device
dev = Device(0)
M, H = 128, 4096
a, w, c = dev.alloc(M * H * 2), dev.alloc(H * H * 2), dev.alloc(M * H * 2)
bias = dev.alloc(H * 2)
dev.fill_synth(a, M * H, 1, 1, 1.0); dev.fill_synth(w, H * H, 1, 2, 1 / 64); dev.fill_synth(bias, H, 1, 3, 0.1)
flush = dev.alloc(256 << 20)
for lay in (1, 0):
  for bn, sk in [(64, 1), (64, 2), (128, 1), (128, 2), (128, 4), (64, 4), (128, 8), (256, 4)]:
    ch = dev.hp_register_chain([dict(kind=1, block_n=bn, a=a, b=w, c=c, bias=0, m=M, n=H, k=H, split_k=sk, b_layout=lay)])
    ms = dev.hp_time_chain(ch, 50)
    print(f"layout={'kblock' if lay == 0 else 'rowmaj'} bn={bn:3d} split={sk}: {ms*1e3:7.2f} us/launch  {32*2**20/(ms*1e-3)/1e9:7.0f} GB/s of W", flush=True)
ch = dev.hp_register_chain([dict(kind=2, block_n=0, a=a, b=0, c=c, bias=bias, m=M, n=H, k=0)])
print(f"bias_gelu: {dev.hp_time_chain(ch, 50)*1e3:.2f} us", flush=True)
dev.close()
