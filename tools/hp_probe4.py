import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2601_04071_b200.device import Device
dev = Device(0)
a = dev.alloc(128 * 8192 * 2); w = dev.alloc(8192 * 8192 * 2); c = dev.alloc(8192 * 8192 * 2)
names = ["prologue", "prod_done", "mma_done", "epi_done", "teardown", "exit_begin", "last", "entry"]
for (n, k, sk) in [(128, 64, 1), (128, 4096, 1), (4096, 4096, 1), (4096, 4096, 4), (4096, 4096, 2)]:
    ch = dev.hp_register_chain([dict(kind=1, block_n=128, a=a, b=w, c=c, bias=0, m=128, n=n, k=k, split_k=sk, b_layout=1)])
    for t in range(3):
        dev.debug_stamps(True)
        dev.hp_launch_direct(ch, dev.hp_next_seq())
        dev.sync()
        d = np.array(dev.debug_stamps(False, 148), dtype=np.float64)
        ncta = max(1, n // 128) * sk
        d = d[:ncta]
        t0 = d[:, 7].min()
        rel = (d - t0) / 1e3
        print(f"n={n} k={k} split={sk} trial {t}: " + "  ".join(f"{nm}={np.nanmedian(np.where(d[:, i] > 0, rel[:, i], np.nan)):.2f}/{np.nanmax(np.where(d[:, i] > 0, rel[:, i], np.nan)):.2f}" for i, nm in enumerate(names)), flush=True)
dev.close()
dev = Device(0)
a = dev.alloc(128 * 8192 * 2); w = dev.alloc(8192 * 8192 * 2); c = dev.alloc(8192 * 8192 * 2)
for (n, k, sk) in [(128, 64, 1), (4096, 4096, 1), (4096, 4096, 2), (4096, 4096, 4), (4096, 4096, 8)]:
    ch = dev.hp_register_chain([dict(kind=1, block_n=128, a=a, b=w, c=c, bias=0, m=128, n=n, k=k, split_k=sk, b_layout=0)])
    print(f"timed n={n} k={k} split={sk}: {dev.hp_time_chain(ch, 50)*1e3:.2f} us", flush=True)
