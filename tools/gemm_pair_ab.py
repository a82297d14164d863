"""In-process A/B: LP GEMM 8192^3 on single CTAs (128x256 tiles, tc_gemm.cuh) vs CTA pairs
(256x256 tiles, cta_group::2, tc_gemm2.cuh); CUDA-event time of full preemptible runs."""
import json
import math
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402

dev = Device(0)
n = 8192
a, b, c = dev.alloc(n * n * 2), dev.alloc(n * n * 2), dev.alloc(n * n * 2)
dev.fill_synth(a, n * n, 1, 1, 1.0)
dev.fill_synth(b, n * n, 1, 2, 1.0 / math.sqrt(n))
os.environ["MS_LP_GEMM_PAIR"] = "0"
k1 = dev.lp_register_gemm(a, b, c, n, n, n)
os.environ["MS_LP_GEMM_PAIR"] = "1"
k2 = dev.lp_register_gemm(a, b, c, n, n, n)
os.environ["MS_LP_GEMM_PAIR"] = "0"
res = {"single": [], "pair": []}
for rnd in range(5):
    for name, k in (("single", k1), ("pair", k2)):
        ms = dev.lp_time_full(k, 4)
        res[name].append(round(2 * n ** 3 / (ms * 1e-3) / 1e12, 1))
print(json.dumps({k: {"median": float(np.median(v)), "runs": v} for k, v in res.items()}))
dev.close()
