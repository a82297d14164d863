"""A/B of the bs=1 decode chain step time alone: this build vs another tree's build
(argv[1] = path of a built tree, e.g. build/r1tree = round-1 commit e1035bc)."""
import os
import sys

tree = sys.argv[1] if len(sys.argv) > 1 else "."
sys.path.insert(0, os.path.abspath(tree))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4  # noqa: E402

dev = Device(0)
w = Config4(dev)
res = {}
for mode in ("1", "0", "1", "0"):
    os.environ["MS_GEMV_DYNAMIC"] = mode
    res.setdefault(mode, []).append(round(min(dev.hp_time_chain(w.chain, 20) for _ in range(3)), 4))
print(tree, res)
dev.close()
