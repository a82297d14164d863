"""In-process A/B of the bs=1 decode chain's consumer layout (MS_GEMV_W, read per launch):
1 warp per ring stage vs 2 warps splitting each unit.  CUDA-event time per decode step.
(The W = 2 kernel was reverted after this A/B — profiles/r01_gemv_w_ab.json,
profiles/r01_gemv_decode.txt — so on the current build both arms run W = 1.)"""
import json
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4  # noqa: E402

dev = Device(0)
c4 = Config4(dev)
res = {"1": [], "2": []}
for rnd in range(5):
    for w in ("1", "2"):
        os.environ["MS_GEMV_W"] = w
        time.sleep(0.1)
        res[w].append(dev.hp_time_chain(c4.chain, 10) * 1e3)
out = {w: {"median_us": float(np.median(v)), "runs_us": [round(x, 1) for x in v]} for w, v in res.items()}
print(json.dumps(out))
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(out, indent=1) + "\n")
dev.close()
