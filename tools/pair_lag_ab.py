"""CTA-pair LP GEMM: MMA queue bound (MS_LP_MMA_LAG, read per launch) vs throughput (best of
10 whole 8192^3 launches) and drain (tools/pair_drain_probe.py phases), alternating settings
in one process.  argv[1:]: lags (default 2 1)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
lags = sys.argv[1:] or ["2", "1"]
out = {}
for rnd in range(2):
    for lag in lags:
        env = dict(os.environ, MS_LP_MMA_LAG=lag)
        code = ("import time,sys; sys.path.insert(0, %r)\n"
                "from paper_2601_04071_b200.device import Device\n"
                "n=8192; d=Device(0); a,b,c=d.alloc(n*n*2),d.alloc(n*n*2),d.alloc(n*n*2)\n"
                "d.fill_synth(a,n*n,1,1,1.0); d.fill_synth(b,n*n,1,2,1/90.5)\n"
                "k=d.lp_register_gemm(a,b,c,n,n,n,block_n=256); best=1e9\n"
                "for _ in range(10):\n time.sleep(0.03); best=min(best,d.lp_time_full(k,1))\n"
                "print(2*n**3/(best*1e-3)/1e12)\n") % str(ROOT)
        tf = float(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                  timeout=300).stdout.strip().splitlines()[-1])
        dr = json.loads(subprocess.run([sys.executable, str(ROOT / "tools" / "pair_drain_probe.py"), "40"], env=env,
                                       capture_output=True, text=True, timeout=300).stdout)
        o = out.setdefault(f"lag={lag}", {"tflops": [], "exit_record_p50_p90_p99": [], "sms_free_p50_p90_p99": [],
                                           "mma_drained_max_p50": [], "epi_done_max_p50": []})
        o["tflops"].append(round(tf, 1))
        o["exit_record_p50_p90_p99"].append(dr["flag_to_exit_record_us"])
        o["sms_free_p50_p90_p99"].append(dr["flag_to_sms_free_us"])
        o["mma_drained_max_p50"].append(dr["phases_us"].get("mma_drained", {}).get("max_p50"))
        o["epi_done_max_p50"].append(dr["phases_us"].get("epi_done", {}).get("max_p50"))
print(json.dumps(out, indent=1))
