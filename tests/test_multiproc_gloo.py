"""N>1 path on CPU: two gloo ranks each run an independent replica scheduler (replay
mode) on their own trace seed; rank results are gathered and aggregated with the same
code bench.py uses for the GPU replicas (no data-path collective)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import json, os, sys
sys.path.insert(0, sys.argv[1])
import torch.distributed as dist
dist.init_process_group("gloo")
rank, ws = dist.get_rank(), dist.get_world_size()
import bench
from paper_2601_04071_b200 import microslice as M, scenarios as S
sc = S.config1(seed=100 + rank, horizon_s=1.0)
r = M.run_scenario(sc, "splitkernel", delays=True)
ex = M.run_scenario(sc, "exclusive")
mine = {"samples": r["delays"], "lp_exit": [], "e2e": [], "rows": [], "ex_rows": [], "kb_rows": [],
        "tiles": float(r["counters"]["lp_work_units"]), "kb_tiles": 1.0,
        "exlp_rate": float(M.run_scenario(sc, "exclusive_lp")["counters"]["lp_work_units"]),
        "slo": {"ttft_ns": 1, "tpot_ns": 1}}
allr = bench.gather(mine, ws)
if rank == 0:
    agg = bench.aggregate_ranks(allr, 1.0)
    print(json.dumps({"p99": bench.percentile(agg["S"], 0.99), "n": len(agg["S"]), "lp_rate": agg["lp_rate"],
                      "per_rank_n": [len(x["samples"]) for x in allr]}))
dist.destroy_process_group()
'''


def test_two_rank_replicas(tmp_path):
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29573")
    procs = [subprocess.Popen([sys.executable, str(w), str(ROOT)], env=dict(env, RANK=str(r), WORLD_SIZE="2"),
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(2)]
    outs = [p.communicate(timeout=240) for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    res = json.loads(outs[0][0].strip().splitlines()[-1])
    sys.path.insert(0, str(ROOT))
    from paper_2601_04071_b200 import microslice as M, scenarios as S
    pooled = []
    for rank in range(2):
        pooled += M.run_scenario(S.config1(seed=100 + rank, horizon_s=1.0), "splitkernel", delays=True)["delays"]
    assert res["n"] == len(pooled) == sum(res["per_rank_n"])
    assert res["p99"] == M.percentile(pooled, 0.99)


def test_config4_leg_pooling():
    """bench.aggregate_config4 pools the per-rank config-4 legs: attainment = sum met / sum
    requests against each rank's own SLO, LP = sum tiles / sum exclusive-LP tiles."""
    sys.path.insert(0, str(ROOT))
    import bench
    row = lambda ttft, tpot, done=True: [0, ttft, tpot, 8, done]  # noqa: E731
    part = lambda slo, ex_rows, split_rows, reef_rows, tiles: {  # noqa: E731
        "slo": {"ttft_ns": slo, "tpot_ns": slo}, "ex_rows": ex_rows, "exlp_tiles": 100, "rate": 9.0, "step_ms": 0.6,
        "splitkernel": {"rows": split_rows, "tiles": tiles[0], "ring": [5000, 7000], "lp_sms": 70.0},
        "reef_req": {"rows": reef_rows, "tiles": tiles[1], "ring": [4000], "lp_sms": 60.0},
        "reef": {"rows": reef_rows, "tiles": tiles[2], "ring": [900000], "lp_sms": 60.0}}
    a = part(10, [row(5, 5), row(9, 9)], [row(5, 5), row(11, 5)], [row(12, 5), row(5, 5, False)], (40, 20, 70))
    b = part(20, [row(5, 5), row(25, 5)], [row(5, 5), row(19, 19)], [row(5, 5), row(5, 5)], (50, 20, 80))
    r = bench.aggregate_config4([a, b])
    assert r["requests"] == 4
    assert r["slo_attainment_exclusive"] == 3 / 4
    assert r["splitkernel"]["slo_attainment"] == 3 / 4
    assert r["reef_req"]["slo_attainment"] == 2 / 4
    assert r["splitkernel"]["lp_throughput_vs_exclusive"] == 90 / 200
    assert r["lp_splitkernel_vs_reef_req"] == (90 / 200) / (40 / 200)
    assert r["reef"]["ring_to_first_hp_cta_p99_us"] == 900.0
