"""CTA-pair LP GEMM 8192^3: the last wave's tile as two 256-column half units
(default) vs one whole tile (MS_LP_PAIR_HALF_TAIL=0), burst (best of 10 launches) and
sustained (S s back to back), alternating rounds in one process (preemptible launches, as
in live runs and the bench's roofline)."""
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
ks = {}
for label, env in (("whole_tail", "0"), ("half_tail", None)):
    if env is None:
        os.environ.pop("MS_LP_PAIR_HALF_TAIL", None)
    else:
        os.environ["MS_LP_PAIR_HALF_TAIL"] = env
    ks[label] = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
os.environ.pop("MS_LP_PAIR_HALF_TAIL", None)
out = {k: {"units": v.total_tiles, "tile_ctas": v.tile_ctas, "burst": [], "sustained": []} for k, v in ks.items()}
import time  # noqa: E402
for rnd in range(6):  # bursts: single launches with idle gaps (clocks recover), variants alternating
    for label, k in ks.items():
        best = 1e9
        for _ in range(5):
            time.sleep(0.05)
            best = min(best, dev.lp_time_full(k, 1))
        out[label]["burst"].append(round(F / (best * 1e-3) / 1e12, 1))
for label, k in ks.items():  # sustained (power-capped), after the bursts
    time.sleep(1.0)
    best = dev.lp_time_full(k, 1)
    reps = max(1, int(S / (best * 1e-3)))
    out[label]["sustained"].append(round(F / (dev.lp_time_full(k, reps) * 1e-3) / 1e12, 1))
print(json.dumps(out))
dev.close()
