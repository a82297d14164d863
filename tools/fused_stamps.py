"""Per-op phase timeline of the fused HP chain kernel (extended debug stamps)."""
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
dev.hp_set_fused(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
ch = dev.hp_register_chain(ops)
info = dev.hp_chain_info(ch)
print(info)
CL = info["cluster"] > 1
big = dev.alloc(256 << 20)
ev = ["p_first_B", "p_A_ready", "p_last_ld", "m_first", "m_commit", "e_tmem", "e_stored", "e_arrived"]
for trial in range(3):
    dev.memset(big, trial, 256 << 20)
    dev.sync()
    dev.debug_stamps(True)
    dev.hp_launch_direct(ch, dev.hp_next_seq())
    dev.sync()
    d = np.array(dev.debug_stamps_ext(148), dtype=np.float64)
    base = np.array(dev.debug_stamps(False, 148), dtype=np.float64) if False else None
    t0 = d[d > 0].min()
    print(f"--- trial {trial} (us from first stamp; median/max over CTAs with units)")
    for oi in range(4):
        cols = []
        for k, nm in enumerate(ev):
            x = d[:128, oi * 8 + k]
            x = x[x > 0]
            cols.append(f"{nm}={np.median(x - t0) / 1e3:6.2f}/{np.max(x - t0) / 1e3:6.2f}" if len(x) else f"{nm}=   -  ")
        extra = ["bar", "red"] if not CL else ["sent", "recvd", "fenced", "barred", "tfenced"]
        for k, nm in enumerate(extra):
            x = d[:148, (40 + oi * 2 + k) if not CL else (40 + oi * 6 + k)]
            x = x[x > 0]
            cols.append(f"{nm}={np.median(x - t0) / 1e3:6.2f}/{np.max(x - t0) / 1e3:6.2f}" if len(x) else f"{nm}=  -  ")
        print(f"op{oi}: " + " ".join(cols))
dev.debug_stamps(False)
print("chain ms (hp_time_chain, 20 reps):", [round(dev.hp_time_chain(ch, 20), 4) for _ in range(3)])
dev.close()
