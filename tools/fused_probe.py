"""Fused vs per-op HP chain timing (config-1 chain: 4 x [128x4096]x[4096x4096]^T + bias/GELU)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
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
big = dev.alloc(256 << 20)
for fused in (0, 2, 1):
    dev.hp_set_fused(fused)
    ch = dev.hp_register_chain(ops)
    print("mode", fused, dev.hp_chain_info(ch))
    print(f"fused={fused} back-to-back: {dev.hp_time_chain(ch, 50)*1e3:.2f} us/chain", flush=True)
    # cold L2: flush between chains (device time of the chain from its own stamps)
    durs = []
    for i in range(20):
        dev.memset(big, i & 0xFF, 256 << 20)
        seq = dev.hp_next_seq()
        dev.hp_launch_direct(ch, seq)
        t = dev.hp_wait(ch, seq, 10)
        durs.append((t["t_done"] - t["t_first_cta"]) / 1e3)
    durs.sort()
    print(f"fused={fused} cold-L2 first-CTA->done: p50 {durs[10]:.2f} max {durs[-1]:.2f} us", flush=True)
if len(sys.argv) > 1:
    names = ["op0_units", "op0_bar", "op0_red", "op1_units", "op1_bar", "exit_begin", "epi_done", "entry"]
    for t in range(3):
        dev.debug_stamps(True)
        dev.hp_launch_direct(ch, dev.hp_next_seq())
        dev.sync()
        d = np.array(dev.debug_stamps(False, 148), dtype=np.float64)[:128]
        t0 = d[:, 7].min()
        rel = (d - t0) / 1e3
        print("  ".join(f"{nm}={np.nanmedian(np.where(d[:, i] > 0, rel[:, i], np.nan)):.2f}/{np.nanmax(np.where(d[:, i] > 0, rel[:, i], np.nan)):.2f}" for i, nm in enumerate(names)), flush=True)
dev.close()
