"""Live memory tier measurements (profiles/r01_tier_probe.json):
  * LP streamer (axpy, 2^28 bf16 = 512 MB per tensor) throughput vs the fraction of its
    chunks spilled to host DRAM (x and y placed by the tier's HBM budget);
  * relocation cost: HP allocations displacing LP chunks (copy to DRAM + VA remap);
  * first-touch allocation cost per chunk per tier.
One GPU on this pool, so the NVLink-peer tier is exercised in replay only."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.tier import MemoryTier  # noqa: E402

CHUNK = 2 << 20


def main():
    out = {"rows": []}
    dev = Device(0)
    n = 1 << 28
    per = 2 * n // CHUNK  # chunks per tensor (256)
    for spill in (0.0, 1 / 16, 1 / 8, 1 / 4, 1 / 2, 1.0):
        local = int(round(2 * per * (1 - spill)))
        tier = MemoryTier(dev, {"hbm_gb": local * CHUNK / 1e9 + 1e-6})
        t0 = time.perf_counter()
        x = tier.alloc(1, 2 * n)
        y = tier.alloc(1, 2 * n)
        t_alloc = time.perf_counter() - t0
        dev.fill_synth(x, n, 1, 1, 1.0)
        dev.fill_synth(y, n, 1, 2, 1.0)
        k = dev.lp_register_axpy(x, y, n, 1.0001)
        ms = dev.lp_time_full(k, 3)
        st = tier.stats()
        row = {"spilled_fraction": st["chunks_dram"] / (2 * per), "chunks_dram": st["chunks_dram"],
               "axpy_ms": ms, "gb_s": 6 * n / (ms * 1e-3) / 1e9, "alloc_ms_per_chunk": t_alloc * 1e3 / (2 * per)}
        print(json.dumps(row), flush=True)
        out["rows"].append(row)
        dev.lp_unregister(k)
        tier.close()
    # relocation cost: fill HBM budget with LP, then an HP allocation displaces 128 chunks
    tier = MemoryTier(dev, {"hbm_gb": 256 * CHUNK / 1e9 + 1e-6})
    x = tier.alloc(1, 256 * CHUNK)
    dev.fill_synth(x, 256 * CHUNK // 2, 1, 3, 1.0)
    t0 = time.perf_counter()
    tier.alloc(0, 128 * CHUNK, high_priority=True)
    dt = time.perf_counter() - t0
    st = tier.stats()
    out["relocation"] = {"chunks": st["relocations"], "ms": dt * 1e3,
                         "gb_s": st["relocated_bytes"] / dt / 1e9, "us_per_chunk": dt * 1e6 / max(1, st["relocations"]),
                         "copy_ms": st["relocate_copy_ns"] / 1e6, "remap_ms": st["relocate_remap_ns"] / 1e6}
    print(json.dumps(out["relocation"]), flush=True)
    tier.close()
    dev.close()
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
