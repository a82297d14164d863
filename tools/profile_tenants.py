"""Profile the LP tenant kernels on B200 into reference KernelSpecs (measured_time) and
their split plans (paper_2601_04071_b200/profiler.py); writes gpurun_out/kernelspecs.json."""
import json
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_04071_b200 import profiler, scenarios  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4  # noqa: E402

dev = Device(0)
w = Config4(dev)
sms = dev.info["sm_count"]
gpu = scenarios.gpu_b200(scenarios.DEFAULT_CALIB)
out = {}
for name, k, resident, tile_bytes in [
        ("lp_gemm_8192", w.lp_gemm, sms - 1, (128 + 256) * 8192 * 2 + 128 * 256 * 2),
        ("lp_axpy_1g", w.lp_axpy, 4 * (sms - 1), 6 * 8192)]:
    spec = profiler.profile_lp_kernel(dev, k, name, resident, tile_bytes)
    plan = profiler.split_plan(gpu, spec)
    plan.pop("slices")
    out[name] = {"kernel_spec": spec, "split_plan": plan}
    print(name, json.dumps(spec["measured_time"]), json.dumps(plan), flush=True)
(ROOT / "gpurun_out" / "kernelspecs.json").write_text(json.dumps(out, indent=1))
dev.close()
