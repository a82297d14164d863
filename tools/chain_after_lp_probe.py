"""Is the bs=1 decode chain slower right after LP work?  Chain duration (first CTA -> done,
device clock) of armed + rung chains: back to back on an idle GPU, right after a full LP
streamer sweep (6 GB), right after a full LP GEMM (8192^3)."""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, Config4  # noqa: E402


def spin(s):
    t = time.perf_counter() + s
    while time.perf_counter() < t:
        pass


dev = Device(0)
c4 = Config4(dev)
c1 = Config1(dev)
res = {}
for rnd in range(3):
    for mode in ("idle", "after_axpy", "after_gemm", "after_axpy_partial"):
        d = []
        for trial in range(12):
            if mode == "after_axpy":
                dev.lp_reset(c4.lp_axpy); dev.lp_run(c4.lp_axpy, 0, c4.lp_axpy.total_tiles); dev.lp_wait(c4.lp_axpy, 30)
            elif mode == "after_axpy_partial":  # ~300 us of streaming, as in a harvested bubble
                dev.lp_reset(c4.lp_axpy); dev.lp_run(c4.lp_axpy, 0, c4.lp_axpy.total_tiles // 3); dev.lp_wait(c4.lp_axpy, 30)
            elif mode == "after_gemm":
                dev.lp_reset(c1.lp); dev.lp_run(c1.lp, 0, c1.lp.total_tiles); dev.lp_wait(c1.lp, 30)
            else:
                spin(300e-6)
            seq = dev.hp_next_seq()
            dev.hp_arm(c4.chain, seq)  # LP work done first: an armed chain's gate holds an SM
            spin(50e-6)
            dev.hp_ring(seq)
            t = dev.hp_wait(c4.chain, seq, 10)
            d.append((t["t_done"] - t["t_first_cta"]) / 1e3)
            dev.sync()
        res.setdefault(mode, []).extend(d)
out = {m: {"p50_us": float(np.percentile(v, 50)), "p90_us": float(np.percentile(v, 90)), "min_us": float(min(v))}
       for m, v in res.items()}
print(json.dumps(out, indent=1))
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(out, indent=1) + "\n")
dev.close()
