"""Development driver: external-tenant session (include/ms_session.h) with a real host
decode loop — config-4 bs=1 decode HP chain per token, a CPU gap U[100,500] us announced
with a hint, LP GEMM + HBM streamer harvesting.  Compares HP step time and LP tiles/s with
the tenant alone and the LP alone."""
import json
import random
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4  # noqa: E402
from paper_2601_04071_b200.session import LiveSession  # noqa: E402


def spin(s):
    t = time.perf_counter() + s
    while time.perf_counter() < t:
        pass


def decode(s, dev, w, tokens, rng, hints):
    steps = []
    for i in range(tokens):
        t0 = time.perf_counter()
        if s:
            t = s.wait(s.submit(w.chain))
        else:
            dev.hp_launch_direct(w.chain, dev.hp_next_seq())
            dev.sync()
        steps.append((time.perf_counter() - t0) * 1e6)
        gap = rng.uniform(100e-6, 500e-6)
        if s and hints and i + 1 < tokens:
            s.hint(300_000)
        spin(gap)
    return steps


dev = Device(0)
w = Config4(dev)
tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 400
rng = random.Random(3)
alone = decode(None, dev, w, tokens, rng, False)
ms_g = dev.lp_time_full(w.lp_gemm, 1)
lp_alone_tps = w.lp_gemm.total_tiles / (ms_g * 1e-3)
res = {"tokens": tokens, "hp_alone_step_us_p50": sorted(alone)[len(alone) // 2]}
for gov in (False, True):
    rng = random.Random(3)
    t0 = time.perf_counter()
    with LiveSession(dev, [w.lp_gemm.id, w.lp_axpy.id], w.chain, {"power_governor": gov}) as s:
        steps = decode(s, dev, w, tokens, rng, True)
    wall = time.perf_counter() - t0
    r = s.report
    key = "governed" if gov else "ungoverned"
    res[key] = {"hp_step_us_p50": sorted(steps)[len(steps) // 2], "hp_step_us_p99": sorted(steps)[int(0.99 * len(steps))],
                "ring_to_first_hp_cta_p99_us": r["ring_to_first_hp_cta"].get("p99_ns", 0) / 1e3,
                "gemm_tiles_per_s_vs_alone": r["lp"][0]["tiles_done"] / wall / lp_alone_tps,
                "lp_launches": r["lp_launches"], "lp_preemptions": r["lp_preemptions"],
                "mean_lp_sms": (r.get("power_governor") or {}).get("mean_lp_sms")}
    print(key, json.dumps(res[key]), flush=True)
print(json.dumps(res))
(ROOT / "gpurun_out" / "session_demo.json").write_text(json.dumps(res, indent=1))
dev.close()
