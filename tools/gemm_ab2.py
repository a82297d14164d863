"""LP GEMM (8192^3 bf16) variants vs cuBLAS, burst (best of 10 single launches) and sustained
(back to back for S s), same process.  Variants: preemptible (pollers on) with MMA-queue lag
2 (default) / unbounded; non-preemptible (no pollers); CTA-pair kernel.  Host-clocked runs
(sync on both sides) for the non-preemptible variants."""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2601_04071_b200.device import Device, lib  # noqa: E402

F = 2 * 8192 ** 3
S = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0


def tf(ms):
    return round(F / (ms * 1e-3) / 1e12, 1)


def cublas():
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    n = max(1, int(S / (best * 1e-3)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        torch.matmul(a, b)
    e1.record(); e1.synchronize()
    return tf(best), tf(e0.elapsed_time(e1) / n)


def ours_preemptible(dev, k):
    best = min(dev.lp_time_full(k, 1) for _ in range(10))
    n = max(1, int(S / (best * 1e-3)))
    return tf(best), tf(dev.lp_time_full(k, n))


def ours_np(dev, k):
    L = lib()
    def run(n):
        dev.sync()
        t = time.perf_counter()
        for _ in range(n):
            L.ms_lp_reset(dev._h, k.id)
            L.ms_lp_run_ex(dev._h, k.id, 0, k.total_tiles, k.total_tiles, 1)
        dev.lp_wait(k, 60)
        dev.sync()
        return (time.perf_counter() - t) / n * 1e3
    run(2)
    best = min(run(1) for _ in range(10))
    n = max(1, int(S / (best * 1e-3)))
    return tf(best), tf(run(n))


torch.cuda.init()
dev = Device(0)
M = N = K = 8192
a, b, c = dev.alloc(M * K * 2), dev.alloc(N * K * 2), dev.alloc(M * N * 2)
dev.fill_synth(a, M * K, 7, 1, 1.0)
dev.fill_synth(b, N * K, 7, 2, 1.0 / 90.5)
k1 = dev.lp_register_gemm(a, b, c, M, N, K, block_n=256)
os.environ["MS_LP_GEMM_PAIR"] = "1"
k2 = dev.lp_register_gemm(a, b, c, M, N, K, block_n=256)
os.environ["MS_LP_GEMM_PAIR"] = "2"
k3 = dev.lp_register_gemm(a, b, c, M, N, K, block_n=256)
del os.environ["MS_LP_GEMM_PAIR"]
out = {}
for rnd in range(2):
    r = {}
    r["cublas"] = cublas(); time.sleep(1)
    r["lag2"] = ours_preemptible(dev, k1); time.sleep(1)
    os.environ["MS_LP_MMA_LAG"] = "0"
    r["lag0"] = ours_preemptible(dev, k1); time.sleep(1)
    r["np_lag0"] = ours_np(dev, k1); time.sleep(1)
    del os.environ["MS_LP_MMA_LAG"]
    r["pair"] = ours_preemptible(dev, k2); time.sleep(1)
    r["pair_np"] = ours_np(dev, k2); time.sleep(1)
    r["pair512"] = ours_preemptible(dev, k3); time.sleep(1)
    os.environ["MS_LP_MMA_LAG"] = "0"
    r["pair512_np"] = ours_np(dev, k3); time.sleep(1)
    dev.set_lp_sm_reserve(0)
    r["pair512_np_74"] = ours_np(dev, k3); time.sleep(1)
    r["np_lag0_148"] = ours_np(dev, k1); time.sleep(1)
    dev.set_lp_sm_reserve(1)
    del os.environ["MS_LP_MMA_LAG"]
    out[f"round{rnd}"] = r
    print(json.dumps({f"round{rnd}": r}), flush=True)
dev.close()
