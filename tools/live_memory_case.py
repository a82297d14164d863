"""Live memory-intensive case on one B200.

Config 4's tenants allocate through the memory tier: HP decode weights pinned in HBM,
LP GEMM + streamer spillable.  The tier's HBM budget is set so that a fraction of the LP
footprint (the streamer's tail chunks, allocated last) lands in host DRAM (no NVLink peer
on this pool).  For each spill fraction: exclusive HP (SLO), exclusive LP, and the
governed split-kernel policy — HP SLO attainment, ring -> first HP CTA p99, LP throughput.
Usage: python tools/live_memory_case.py [horizon_s] [out.json]"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4, live_run  # noqa: E402
from paper_2601_04071_b200.tier import MemoryTier  # noqa: E402
from tools.live_check import brief  # noqa: E402

CHUNK = 2 << 20


def main():
    horizon = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
    out = {"horizon_s": horizon, "rows": []}
    dev = Device(0)
    hp_bytes = 2 * (16 * (3072 * 2048 + 2048 * 2048 + 16384 * 2048 + 2048 * 8192) + 128256 * 2048)
    hp_chunks = -(-hp_bytes // CHUNK) + 32  # + activation buffers (one chunk each)
    lp_chunks = 3 * (8192 * 8192 * 2 // CHUNK) + 2 * ((1 << 30) * 2 // CHUNK)
    cases = [(0.0, 8), (0.02, 0), (0.02, 8), (0.125, 8), (0.125, 2)]  # (spill, slow-tile admission; 0 = off)
    for spill, slow_max in cases:
        budget = (hp_chunks + int(lp_chunks * (1 - spill))) * CHUNK
        tier = MemoryTier(dev, {"hbm_gb": budget / 1e9 + 1e-6})
        w = Config4(dev, tier=tier, slow_max=slow_max)
        st = tier.stats()
        time.sleep(0.5)
        calib = w.calibrate()
        sc = w.scenario(seed=1, horizon_s=horizon, rate=w.hp_rate(0.8))
        ex = live_run(dev, sc, "exclusive", w.binding(), w.options())
        slo = {"ttft_ns": ex["own_p99"]["ttft_ns"], "tpot_ns": ex["own_p99"]["tpot_ns"]}
        ex2 = live_run(dev, sc, "exclusive", w.binding(), w.options(slo=slo))
        exlp = live_run(dev, sc, "exclusive_lp", w.binding(), w.options())
        row = {"spill_target": spill, "slow_max": slow_max, "chunks_dram": st["chunks_dram"], "chunks_local": st["chunks_local"],
               "lp_dram_fraction": st["chunks_dram"] / lp_chunks, "calib": calib,
               "slo_attainment_exclusive": ex2.get("slo_attainment")}
        for pol, kw in (("splitkernel", {"power_governor": True}), ("reef_req", {"power_governor": True})):
            r = live_run(dev, sc, pol, w.binding(), w.options(slo=slo, **kw))
            b = brief(r)
            b["lp_norm"] = r["lp"]["tiles_per_s"] / max(1e-9, exlp["lp"]["tiles_per_s"])
            row[pol] = b
        print(json.dumps(row), flush=True)
        out["rows"].append(row)
        dev.sync()
        dev.lp_unregister(w.lp_gemm)
        dev.lp_unregister(w.lp_axpy)
        dev.hp_unregister_chain(w.chain)
        tier.close()
    dev.close()
    if len(sys.argv) > 2:
        Path(sys.argv[2]).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
