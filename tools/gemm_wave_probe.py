"""CTA-pair LP GEMM 8192^3 wave quantisation probe: burst time (best of 7 single launches
with idle gaps) of the unit ranges [0, w * pairs) for w = 1 .. 7 and of the whole grid
(512 units = 7 waves of 73 pairs + 1 unit), with the tail tile whole, as halves and as quarters."""
import json
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device  # noqa: E402

n = 8192
dev = Device(0)
a, b, c = dev.alloc(n * n * 2), dev.alloc(n * n * 2), dev.alloc(n * n * 2)
dev.fill_synth(a, n * n, 1, 1, 1.0)
dev.fill_synth(b, n * n, 1, 2, 1.0 / 90.5)
os.environ["MS_LP_PAIR_HALF_TAIL"] = "0"
kw = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
os.environ.pop("MS_LP_PAIR_HALF_TAIL", None)
os.environ["MS_LP_PAIR_TAIL_PARTS"] = "2"
kh = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
os.environ.pop("MS_LP_PAIR_TAIL_PARTS", None)
kq = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 73


def best(k, lo, hi, reps=7):
    t = 1e9
    for _ in range(reps):
        time.sleep(0.03)
        t = min(t, dev.lp_time_range(k, lo, hi, 1))
    return t


out = {"pairs_assumed": pairs, "units_whole": kw.total_tiles, "units_half": kh.total_tiles,
       "units_quarter": kq.total_tiles, "ranges_ms": {}}
for w in range(1, 8):
    out["ranges_ms"][f"[0,{w * pairs})"] = round(best(kw, 0, w * pairs), 4)
out["ranges_ms"]["whole_tail_full"] = round(best(kw, 0, kw.total_tiles), 4)
out["ranges_ms"]["half_tail_full"] = round(best(kh, 0, kh.total_tiles), 4)
out["ranges_ms"]["quarter_tail_full"] = round(best(kq, 0, kq.total_tiles), 4)
for rnd in range(3):  # alternating repeats of the three whole-grid variants
    for lab, kk in (("whole", kw), ("half", kh), ("quarter", kq)):
        out["ranges_ms"].setdefault(f"{lab}_repeats", []).append(round(best(kk, 0, kk.total_tiles, 5), 4))
F = 2 * n ** 3
out["tflops_whole"] = round(F / (out["ranges_ms"]["whole_tail_full"] * 1e-3) / 1e12, 1)
out["tflops_half"] = round(F / (out["ranges_ms"]["half_tail_full"] * 1e-3) / 1e12, 1)
out["tflops_quarter"] = round(F / (out["ranges_ms"]["quarter_tail_full"] * 1e-3) / 1e12, 1)
print(json.dumps(out, indent=1))
dev.close()
