"""Fixed vs proportional cost of the tcgen05 GEMM kernel (diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device
dev = Device(0)
a = dev.alloc(128 * 8192 * 2); w = dev.alloc(8192 * 8192 * 2); c = dev.alloc(8192 * 8192 * 2)
dev.fill_synth(a, 128 * 8192, 1, 1, 1.0); dev.fill_synth(w, 8192 * 8192, 1, 2, 1 / 64)
for (m, n, k, bn, sk) in [(128, 128, 64, 128, 1), (128, 128, 4096, 128, 1), (128, 4096, 64, 128, 1),
                          (128, 4096, 512, 128, 1), (128, 4096, 4096, 128, 1), (128, 4096, 4096, 128, 4),
                          (128, 1024, 4096, 128, 1), (128, 8192, 4096, 128, 1), (128, 4096, 8192, 128, 1)]:
    ch = dev.hp_register_chain([dict(kind=1, block_n=bn, a=a, b=w, c=c, bias=0, m=m, n=n, k=k, split_k=sk, b_layout=1)])
    ms = dev.hp_time_chain(ch, 30)
    print(f"m={m} n={n:5d} k={k:5d} bn={bn} split={sk}: {ms*1e3:8.2f} us", flush=True)
k = dev.lp_register_gemm(a, w, c, 128, 4096, 4096, block_n=128)
print("LP-path same GEMM (preemptible run):", dev.lp_time_full(k, 20) * 1e3, "us")
dev.close()
