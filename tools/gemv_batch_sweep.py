"""Decode-chain step time alone (CUDA events, best of 3 x 20 launches): static unit plan vs
dynamic claiming with claim batches B (MS_GEMV_CLAIM_BATCH)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4  # noqa: E402

dev = Device(0)
w = Config4(dev)
res = {}
for dyn, b in (("0", "1"), ("1", "4"), ("1", "16"), ("1", "64"), ("1", "256"), ("0", "1")):
    os.environ["MS_GEMV_DYNAMIC"], os.environ["MS_GEMV_CLAIM_BATCH"] = dyn, b
    res.setdefault(f"dyn={dyn} B={b}", []).append(round(min(dev.hp_time_chain(w.chain, 20) for _ in range(3)), 4))
print(res)
dev.close()
