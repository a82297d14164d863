"""A/B: the LP tcgen05 GEMM (8192^3 bf16) vs cuBLAS (torch.matmul) measured the way
MEASURED_PEAKS.json measures the peak: best of 10 single launches (burst) and back to back
for ~4 s (sustained), CUDA events, same process, same box.  Prints one JSON line."""
import json
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2601_04071_b200.live import Config1  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402

F = 2 * 8192 ** 3
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0


def cublas():
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    n = max(1, int(secs / (best * 1e-3)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        torch.matmul(a, b)
    e1.record()
    e1.synchronize()
    sus = e0.elapsed_time(e1) / n
    del a, b
    torch.cuda.empty_cache()
    return best, sus


def ours(dev, w):
    best = min(dev.lp_time_full(w.lp, 1) for _ in range(10))
    n = max(1, int(secs / (best * 1e-3)))
    sus = dev.lp_time_full(w.lp, n)
    return best, sus


torch.cuda.init()
dev = Device(0)
w = Config1(dev)
out = {}
for rnd in range(2):
    cb, cs = cublas()
    time.sleep(2.0)
    ob, os_ = ours(dev, w)
    time.sleep(2.0)
    out[f"round{rnd}"] = {"cublas_burst_tflops": F / (cb * 1e-3) / 1e12, "cublas_sustained_tflops": F / (cs * 1e-3) / 1e12,
                          "ours_burst_tflops": F / (ob * 1e-3) / 1e12, "ours_sustained_tflops": F / (os_ * 1e-3) / 1e12}
print(json.dumps(out), flush=True)
dev.close()
