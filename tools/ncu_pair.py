"""ncu target: the LP GEMM 8192^3 on CTA pairs (MS_LP_GEMM_PAIR=1) and single-CTA, two runs
each, non-preemptible and preemptible."""
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_04071_b200.device import Device, lib  # noqa: E402

dev = Device(0)
M = N = K = 8192
a, b, c = dev.alloc(M * K * 2), dev.alloc(N * K * 2), dev.alloc(M * N * 2)
dev.fill_synth(a, M * K, 7, 1, 1.0)
dev.fill_synth(b, N * K, 7, 2, 1.0 / 90.5)
os.environ["MS_LP_GEMM_PAIR"] = "1"
k2 = dev.lp_register_gemm(a, b, c, M, N, K, block_n=256)
del os.environ["MS_LP_GEMM_PAIR"]
k1 = dev.lp_register_gemm(a, b, c, M, N, K, block_n=256)
L = lib()
for k in (k2, k1):
    for _ in range(2):
        L.ms_lp_reset(dev._h, k.id)
        L.ms_lp_run_ex(dev._h, k.id, 0, k.total_tiles, k.total_tiles, 1)
        dev.lp_wait(k, 60)
dev.close()
print("done")
