"""Does a parked HP gate keep a CTA pair of the LP GEMM off its SM?  Times the full 8192^3
pair GEMM (non-preemptible) on 74 pairs (LP SM reserve 0) and 73 pairs (reserve 1 -> one
TPC) without a gate and with an armed, unrung config-1 chain gate.  74 pairs + a parked gate:
waits 2 s for the run; if it has not finished, rings the gate and reports the run as blocked
until the ring."""
import json
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_04071_b200.device import Device, DeviceError, lib  # noqa: E402
from paper_2601_04071_b200.live import Config1  # noqa: E402

dev = Device(0)
w = Config1(dev)
L = lib()
k = w.lp


def t_full(n=5):
    # (no device-wide sync: it would wait for the parked gate)
    t = time.perf_counter()
    for _ in range(n):
        L.ms_lp_reset(dev._h, k.id)
        L.ms_lp_run_ex(dev._h, k.id, 0, k.total_tiles, k.total_tiles, 1)
        dev.lp_wait(k, 20)
    return round((time.perf_counter() - t) / n * 1e3, 4)


out = {"tile_ctas": k.tile_ctas, "tiles": k.total_tiles}
for reserve in (0, 1):
    dev.set_lp_sm_reserve(reserve)
    t_full(2)
    out[f"reserve{reserve}_nogate_ms"] = t_full()
dev.set_lp_sm_reserve(1)
seq = dev.hp_next_seq()
dev.hp_arm(w.chain, seq)
time.sleep(0.01)
out["reserve1_gate_ms"] = t_full()
dev.hp_ring(seq)
dev.hp_wait(w.chain, seq, 10)
dev.sync()
seq = dev.hp_next_seq()
dev.hp_arm(w.chain, seq)
time.sleep(0.01)
dev.set_lp_sm_reserve(0)
L.ms_lp_reset(dev._h, k.id)
L.ms_lp_run_ex(dev._h, k.id, 0, k.total_tiles, k.total_tiles, 1)
try:
    dev.lp_wait(k, 2)
    out["reserve0_gate"] = "completed with the gate parked"
except DeviceError:
    out["reserve0_gate"] = "blocked until the gate was rung"
dev.hp_ring(seq)
dev.hp_wait(w.chain, seq, 10)
dev.lp_wait(k, 60)
print(json.dumps(out), flush=True)
dev.set_lp_sm_reserve(1)
dev.close()
