"""Is the fused HP chain's mainloop bound by the chip's TMA/L2 delivery rate or by each SM's
ingest?  4-op chains [128 x 4096] x [4096 x N]^T with N = 4096 / 2048 / 1024 (32 / 16 / 8
column tiles x 4 k-slices = 128 / 64 / 32 CTAs, same 512 KB per CTA per op): chip-bound ->
the mainloop shrinks with N; SM-bound -> it stays.  Per-op phase stamps as fused_stamps.py."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402

dev = Device(0)
M, K = 128, 4096
x = dev.alloc(M * K * 2)
dev.fill_synth(x, M * K, 1, 100, 1.0)
big = dev.alloc(256 << 20)
out = {}
for N in (4096, 2048, 1024):
    ws = [dev.alloc(N * K * 2) for _ in range(4)]
    ys = [dev.alloc(M * N * 2) for _ in range(4)]
    for i, w in enumerate(ws):
        dev.fill_synth(w, N * K, 1, 101 + i, 1.0 / 64)
    ops = [dict(kind=1, block_n=128, a=x, b=ws[i], c=ys[i], bias=0, m=M, n=N, k=K, split_k=4) for i in range(4)]
    ch = dev.hp_register_chain(ops)
    info = dev.hp_chain_info(ch)
    ml, ex = [], []
    for trial in range(4):
        dev.memset(big, trial, 256 << 20)
        dev.sync()
        dev.debug_stamps(True)
        dev.hp_launch_direct(ch, dev.hp_next_seq())
        dev.sync()
        d = np.array(dev.debug_stamps_ext(148), dtype=np.float64)
        g = info["fused_grid"]
        for oi in range(1, 4):   # ops 1-3 (weights L2-prefetched during the previous op)
            mf, mc = d[:g, oi * 8 + 3], d[:g, oi * 8 + 4]
            ok = (mf > 0) & (mc > 0)
            ml.append(float(np.median(mc[ok] - mf[ok])) / 1e3)
    dev.debug_stamps(False)
    t = [round(dev.hp_time_chain(ch, 20) * 1e3, 2) for _ in range(3)]
    out[N] = {"grid": info["fused_grid"], "cluster": info["cluster"], "mainloop_us_median": round(float(np.median(ml)), 2),
              "chain_us": t, "weights_mb_per_op": N * K * 2 / 1e6}
    print(N, out[N], flush=True)
    dev.hp_unregister_chain(ch)
    for p in ws + ys:
        dev.free(p)
print(json.dumps(out))
dev.close()
