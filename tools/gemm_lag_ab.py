"""CTA-pair LP GEMM (8192^3, preemptible launch as in live runs): MMA-queue bound
MS_LP_MMA_LAG 2 (default) vs 1 vs 0 (unbounded), burst (best of 10) and sustained (S s),
alternating rounds in one process."""
import json
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device  # noqa: E402

F = 2 * 8192 ** 3
S = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
dev = Device(0)
n = 8192
a, b, c = dev.alloc(n * n * 2), dev.alloc(n * n * 2), dev.alloc(n * n * 2)
dev.fill_synth(a, n * n, 1, 1, 1.0)
dev.fill_synth(b, n * n, 1, 2, 1.0 / 90.5)
k = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
assert k.tile_ctas == 2
out = {}
for rnd in range(3):
    for lag in ("2", "1", "0"):
        os.environ["MS_LP_MMA_LAG"] = lag
        dev.lp_time_full(k, 3)
        best = min(dev.lp_time_full(k, 1) for _ in range(10))
        reps = max(1, int(S / (best * 1e-3)))
        sus = dev.lp_time_full(k, reps)
        out.setdefault(lag, []).append((round(F / (best * 1e-3) / 1e12, 1), round(F / (sus * 1e-3) / 1e12, 1)))
print(json.dumps(out))
dev.close()
