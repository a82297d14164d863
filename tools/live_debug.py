import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device
from paper_2601_04071_b200.live import Config1, live_run
dev = Device(0)
w = Config1(dev)
w.calibrate(2)
import os
if os.environ.get("RESERVE"): dev.set_lp_sm_reserve(int(os.environ["RESERVE"]))
r = live_run(dev, w.scenario(seed=3, horizon_s=1.0), "splitkernel", w.binding(), w.options(debug_stamps=40))
names = ["seen", "prod_done", "mma_done", "epi_done", "teardown", "exit_begin", "last"]
print("flag->last exit", r["preempt_flag_to_last_lp_exit"])
for run in r["debug_phases"][5:20]:
    print("  ".join(f"{n}:{'/'.join(str(round(x/1e3,1)) for x in ph)}" for n, ph in zip(names, run[:7])), "late", run[7], "counts", run[8])
