"""Memory-intensive case in replay.

Config 4's tenants on one B200 of an HGX node with footprints that overflow HBM (HP
60 GB pinned, LP 150 GB -> ~30 GB spilled to NVLink peers / DRAM).  Compares eviction
policies (contention-first vs round-robin) and sharing policies, plus the no-spill
reference point.  Usage: python tools/memory_case.py [horizon_s] [out.json]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200 import microslice as M  # noqa: E402
from paper_2601_04071_b200 import scenarios as S  # noqa: E402


RATE = float(sys.argv[3]) if len(sys.argv) > 3 else 10.0


def row(sc, pol):
    t = time.time()
    r = M.run_scenario(sc, pol, report=True)["report"]
    return {"slo_attainment": r["hp"]["slo_attainment"], "lp_throughput_normalized": r["lp"]["throughput_normalized"],
            "preempt_p99_ns": r["hp"]["preemption"]["p99_ns"], "ttft_p99_ns": r["hp"]["ttft_p99_ns"],
            "tpot_p99_ns": r["hp"]["tpot_p99_ns"], "wall_s": round(time.time() - t, 2)}


def main():
    horizon = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
    out = {"workload": "config 4 tenants, HP 60 GB pinned + LP 90+60 GB on a 180 GB B200, 7 NVLink-5 peers "
                       "(900 GB/s, 2 us; peers 1 and 4 carry 600 / 300 GB/s background), 40 GB free each",
           "horizon_s": horizon, "rate_req_s": RATE, "rows": {}}
    cases = {"contention_first": S.config_memory(seed=1, horizon_s=horizon, rate=RATE),
             "round_robin": S.config_memory(seed=1, horizon_s=horizon, rate=RATE, eviction="round_robin"),
             "dram_only (no free peer memory)": S.config_memory(seed=1, horizon_s=horizon, rate=RATE, peer_free_gb=(0.0,) * 7),
             "no_spill (LP fits: 100 GB)": S.config_memory(seed=1, horizon_s=horizon, rate=RATE, lp_gb=(60.0, 40.0))}
    for name, sc in cases.items():
        out["rows"][name] = {pol: row(sc, pol) for pol in ("splitkernel", "reef", "spatial")}
        print(name, json.dumps(out["rows"][name]), flush=True)
    if len(sys.argv) > 2:
        Path(sys.argv[2]).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
