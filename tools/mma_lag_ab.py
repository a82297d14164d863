"""In-process A/B of the LP GEMM MMA queue bound (MS_LP_MMA_LAG, read per launch):
CUDA-event time of full preemptible 8192^3 runs, alternating settings, plus the
flag -> last LP exit latency of preempted runs per setting."""
import json
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1  # noqa: E402


def spin(s):
    t = time.perf_counter() + s
    while time.perf_counter() < t:
        pass


dev = Device(0)
c1 = Config1(dev)
k = c1.lp
res = {}
for rnd in range(4):
    for lag in ("0", "2", "1", "4"):
        os.environ["MS_LP_MMA_LAG"] = lag
        ms = dev.lp_time_full(k, 4)
        res.setdefault(lag, {"tflops": [], "exit": []})["tflops"].append(2 * 8192 ** 3 / (ms * 1e-3) / 1e12)
for lag in ("0", "2", "1", "4"):
    os.environ["MS_LP_MMA_LAG"] = lag
    off, _ = dev.calibrate(100)
    for trial in range(30):
        dev.lp_reset(k)
        dev.lp_run(k, 0, k.total_tiles)
        spin(200e-6 + 1e-5 * (trial % 7))
        _, t_raise = dev.preempt_raise()
        st = dev.lp_wait(k, 30)
        if st["preempted"]:
            res[lag]["exit"].append((st["t_exit"] - off - t_raise) / 1e3)
out = {lag: {"tflops_median": float(np.median(v["tflops"])), "tflops": [round(x, 1) for x in v["tflops"]],
             "exit_p50_us": float(np.percentile(v["exit"], 50)), "exit_p90_us": float(np.percentile(v["exit"], 90)),
             "exit_p99_us": float(np.percentile(v["exit"], 99))} for lag, v in res.items()}
print(json.dumps(out, indent=1))
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(out, indent=1) + "\n")
dev.close()
