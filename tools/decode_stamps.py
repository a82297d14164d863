"""Per-op timeline of the first decode layer of the config-4 fused HP chain (diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2601_04071_b200.device import Device
from paper_2601_04071_b200.live import Config4

dev = Device(0)
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dev.hp_set_fused(mode)
w = Config4(dev)
print("chain info", dev.hp_chain_info(w.chain), "step ms", dev.hp_time_chain(w.chain, 5))
ev = ["p_first_B", "p_A_ready", "p_last_ld", "m_first", "m_commit", "e_tmem", "e_stored", "e_arrived"]
names = ["qkv", "o", "gu", "silu", "down"]
for trial in range(2):
    dev.debug_stamps(True)
    seq = dev.hp_next_seq()
    dev.hp_launch_direct(w.chain, seq)
    tm = dev.hp_wait(w.chain, seq, 10)
    d = np.array(dev.debug_stamps_ext(148), dtype=np.float64)
    t0 = tm["t_first_cta"]
    print(f"--- trial {trial}: step {(tm['t_done'] - t0) / 1e3:.1f} us")
    for oi in range(5):
        cols = []
        for k, nm in enumerate(ev):
            x = d[:, oi * 8 + k]
            x = x[x > 0]
            cols.append(f"{nm}={np.median(x - t0) / 1e3:6.1f}/{np.max(x - t0) / 1e3:6.1f}" if len(x) else f"{nm}=   -  ")
        print(f"{names[oi]:5s}: " + " ".join(cols))
dev.close()
