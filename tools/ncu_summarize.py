"""Summarise ncu --set full captures (gpurun_out/r02/prof_*.ncu-rep) into a JSON of the
per-launch numbers the roofline needs: duration, DRAM bytes read + written (traffic), DRAM
throughput %, tensor-pipe active %, SM throughput %, registers.  Usage:
    python tools/ncu_summarize.py gpurun_out/r02 > profiles/r02_ncu_summary.json"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    hdr, units = r[0], r[1]
    res = []
    for line in r[2:]:
        d = {"kernel": line[hdr.index("Kernel Name")][:90]}
        for m, k in WANT.items():
            if m in hdr:
                v = line[hdr.index(m)].replace(",", "")
                try:
                    d[k] = float(v)
                except ValueError:
                    d[k] = v
                d[k + "_unit"] = units[hdr.index(m)]
        res.append(d)
    return res


src = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/r02")
print(json.dumps({rep.stem: rows(rep) for rep in sorted(src.glob("*.ncu-rep"))}, indent=1))
