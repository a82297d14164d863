"""ncu target: one cuBLAS 8192^3 bf16 GEMM (torch.matmul) and one LP tcgen05 GEMM of the same
shape, back to back (capture both with -k regex and compare the raw pages)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2601_04071_b200.live import Config1  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402

a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
dev = Device(0)
w = Config1(dev)
for _ in range(2):
    dev.lp_run(w.lp, 0, w.lp.total_tiles)
    dev.lp_wait(w.lp, 60)
dev.close()
print("done")
