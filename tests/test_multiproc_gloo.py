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
sc = S.config1(seed=100 + rank, horizon_s=float(sys.argv[2]))
r = M.run_scenario(sc, "splitkernel", delays=True)
exlp = float(M.run_scenario(sc, "exclusive_lp")["counters"]["lp_work_units"])
kb = {p: {"rows": [], "tiles": 1.0, "samples": []} for p in ("reef", "reef_req")}
mine = {"samples": r["delays"], "inflight": r["delays"], "idle": [], "lp_exit": [], "e2e": [], "rows": [],
        "ex_rows": [], "kb": kb, "pb": {"rows": [], "tiles": 0.0, "samples": [], "inflight": [], "gov": []},
        "tiles": float(r["counters"]["lp_work_units"]), "exlp_rate": exlp, "slo": {"ttft_ns": 1, "tpot_ns": 1}}
allr = bench.gather(mine, ws)
bench.barrier(ws)
if rank == 0:
    agg = bench.aggregate_ranks(allr, 1.0, 1.0)
    print(json.dumps({"p99": bench.percentile(agg["S"], 0.99), "n": len(agg["S"]), "lp_rate": agg["lp_rate"],
                      "ex_rate": agg["ex_rate"], "per_rank_n": [len(x["samples"]) for x in allr],
                      "backend": dist.get_backend()}))
dist.destroy_process_group()
'''


def _run(tmp_path, ws, port, horizon):
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    procs = [subprocess.Popen([sys.executable, str(w), str(ROOT), str(horizon)],
                              env=dict(env, RANK=str(r), WORLD_SIZE=str(ws)),
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(ws)]
    outs = [p.communicate(timeout=400) for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    res = json.loads(outs[0][0].strip().splitlines()[-1])
    sys.path.insert(0, str(ROOT))
    from paper_2601_04071_b200 import microslice as M, scenarios as S
    pooled, lp, ex = [], 0.0, 0.0
    for rank in range(ws):
        sc = S.config1(seed=100 + rank, horizon_s=horizon)
        r = M.run_scenario(sc, "splitkernel", delays=True)
        pooled += r["delays"]
        lp += float(r["counters"]["lp_work_units"])
        ex += float(M.run_scenario(sc, "exclusive_lp")["counters"]["lp_work_units"])
    assert res["backend"] == "gloo"  # replicas: host plumbing only, never NCCL
    assert res["n"] == len(pooled) == sum(res["per_rank_n"])
    assert res["p99"] == M.percentile(pooled, 0.99)
    assert abs(res["lp_rate"] - lp) < 1e-6 and abs(res["ex_rate"] - ex) < 1e-6


def test_two_rank_replicas(tmp_path):
    _run(tmp_path, 2, 29573, 1.0)


def test_eight_rank_replicas(tmp_path):
    """Config 5 shape: 8 independent replica schedulers (one per GPU of an 8xB200 node),
    each on its own trace seed, aggregated on rank 0 over gloo."""
    _run(tmp_path, 8, 29574, 0.5)


def test_policy_leg_pooling():
    """bench.aggregate_leg pools the per-rank config legs: attainment = sum met / sum
    requests against each rank's own SLO, LP = sum rate / sum exclusive-LP rate."""
    sys.path.insert(0, str(ROOT))
    import bench
    row = lambda ttft, tpot, done=True: [0, ttft, tpot, 8, done]  # noqa: E731
    pol = lambda rows, rate, ring, infl: {"rows": rows, "tiles_per_s": rate, "ring": ring, "inflight": infl,  # noqa: E731
                                          "lp_exit": [8000], "step_p50_us": 550.0, "lp_sms": 70.0}
    part = lambda slo, ex_rows, split_rows, reef_rows, rates: {  # noqa: E731
        "slo": {"ttft_ns": slo, "tpot_ns": slo}, "ex_rows": ex_rows, "exlp_rate": 100.0, "rate": 9.0,
        "ex_step_p50_us": 549.0,
        "splitkernel": pol(split_rows, rates[0], [5000, 7000], [7000]),
        "reef_req": pol(reef_rows, rates[1], [4000], []),
        "reef": pol(reef_rows, rates[2], [900000], [])}
    a = part(10, [row(5, 5), row(9, 9)], [row(5, 5), row(11, 5)], [row(12, 5), row(5, 5, False)], (40, 20, 70))
    b = part(20, [row(5, 5), row(25, 5)], [row(5, 5), row(19, 19)], [row(5, 5), row(5, 5)], (50, 20, 80))
    r = bench.aggregate_leg([a, b], "test")
    assert r["requests"] == 4
    assert r["slo_attainment_exclusive"] == 3 / 4
    assert r["splitkernel"]["slo_attainment"] == 3 / 4
    assert r["reef_req"]["slo_attainment"] == 2 / 4
    assert r["splitkernel"]["lp_throughput_vs_exclusive"] == 90 / 200
    assert r["lp_splitkernel_vs_reef_req"] == round((90 / 200) / (40 / 200), 3)
    assert r["reef"]["ring_to_first_hp_cta_p99_us"] == 900.0
    assert r["splitkernel"]["preempt_lp_in_flight_p99_us"] == 7.0
    assert r["targets"] == {"p99_le_10us": True, "slo_within_1pt": True, "lp_ge_2x_kernel_boundary": True}


def test_host_facts():
    sys.path.insert(0, str(ROOT))
    import bench
    h = bench.host_info()
    assert h["nproc"] >= 1 and h["cpu_model"]
    assert isinstance(bench.numa_core_for(0), int)  # -1 without a GPU / NVML
