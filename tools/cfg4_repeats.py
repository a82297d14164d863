"""Config-4 leg repeated (bench.py run_policy_leg, 32 s = 2 interleaved windows per repeat,
different trace seeds), to show the run-to-run spread of the p99-based SLO attainment and
of the LP ratio vs the request-level kernel boundary.  Optional argv[1]: MS_LP_GEMM_PAIR for
the LP GEMM (default: the kernel bench.py uses)."""
import json
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
if len(sys.argv) > 1:
    os.environ["MS_LP_GEMM_PAIR"] = sys.argv[1]
import bench  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4  # noqa: E402

dev = Device(0)
w4 = Config4(dev)
w4.calibrate()
reps = int(os.environ.get("REPS", "3"))
out = []
for r in range(reps):
    leg = bench.run_policy_leg(dev, w4, 32.0, 7 + 1000 * r, w4.hp_rate(0.8), reef_s=8.0)
    agg = bench.aggregate_leg([leg], "cfg4")
    sk = agg["splitkernel"]
    row = {"seed": 7 + 1000 * r, "requests": agg["requests"], "slo_exclusive": agg["slo_attainment_exclusive"],
           "slo_splitkernel": sk["slo_attainment"], "slo_reef_req": agg["reef_req"]["slo_attainment"],
           "lp_vs_reef_req": agg["lp_splitkernel_vs_reef_req"], "lp_vs_exclusive": sk["lp_throughput_vs_exclusive"],
           "step_p50_ex_us": agg["exclusive_step_p50_us"], "step_p50_sk_us": sk["hp_step_p50_us"],
           "inflight_p99_us": sk["preempt_lp_in_flight_p99_us"], "lp_exit_p99_us": sk["flag_to_last_lp_exit_p99_us"],
           "mean_lp_sms": sk["mean_lp_sms"]}
    print(json.dumps(row), flush=True)
    out.append(row)
json.dump(out, open(os.environ.get("OUT", "gpurun_out/cfg4_repeats.json"), "w"), indent=1)
dev.close()
