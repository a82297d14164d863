"""LP GEMM raster sweep: CUDA-event time of the 8192^3 persistent tcgen05 GEMM for several
group-M raster widths (tile order: group_m M-tiles x all N-tiles per group)."""
import json
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_04071_b200.device import Device  # noqa: E402


def main():
    dev = Device(0)
    n = 8192
    a, b, c = dev.alloc(n * n * 2), dev.alloc(n * n * 2), dev.alloc(n * n * 2)
    dev.fill_synth(a, n * n, 1, 1, 1.0)
    dev.fill_synth(b, n * n, 1, 2, 1.0 / math.sqrt(n))
    rows = []
    for rep in range(2):
        for g in (4, 8, 12, 16, 24, 32, 64):
            k = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256, group_m=g)
            time.sleep(0.2)
            ms = dev.lp_time_full(k, 5)
            dev.lp_unregister(k)
            row = {"rep": rep, "group_m": g, "ms": ms, "tflops": 2 * n ** 3 / (ms * 1e-3) / 1e12}
            print(json.dumps(row), flush=True)
            rows.append(row)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(rows, indent=1) + "\n")
    dev.close()


if __name__ == "__main__":
    main()
