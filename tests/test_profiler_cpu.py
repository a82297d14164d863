"""Profiler output (paper_2601_04071_b200/profiler.py) on CPU: the KernelSpec it builds
from measured rows parses in the reference schema, reproduces the persistent kernel's
residency through Eq. 1, interpolates the measured rows, and yields a valid split plan."""
import math

from paper_2601_04071_b200 import microslice as M, profiler, scenarios

GPU = scenarios.gpu_b200(scenarios.DEFAULT_CALIB)


def test_sweep_points():
    assert profiler.sweep_points(1024, 147) == [73, 147, 294, 588, 1024]
    pts = profiler.sweep_points(131072, 588)
    assert pts[0] == 294 and pts[-1] == 131072 and pts == sorted(set(pts))
    assert profiler.sweep_points(100, 147) == [73, 100]


def test_kernel_spec_roundtrip_and_split_plan():
    rows = [(73, 69_621), (147, 72_320), (294, 127_093), (588, 248_864), (1176, 498_421), (2048, 863_605)]
    spec = profiler.kernel_spec("lp_gemm_8192", 2048, 147, 148, (128 + 256) * 8192 * 2 + 128 * 256 * 2, rows)
    assert M.concurrent_capacity(GPU, spec) == 148  # 1 persistent CTA per SM
    norm = M.normalize_scenario({"name": "p", "seed": 1, "horizon": {"value": 1, "unit": "ms"}, "gpu": GPU,
                                 "kernels": [spec], "tasks": [], "traces": []})
    k = norm["kernels"][0]
    assert [(r["n_blocks"], r["time"]["value"]) for r in k["measured_time"]] == rows
    plan = profiler.split_plan(GPU, spec, cap_ns=200_000)
    assert plan["blocks_per_slice"] >= 1 and plan["predicted_slice_time"] <= 200_000
    assert sum(math.prod(s[3:6]) for s in plan["slices"]) == 2048
    # the measured oracle, not the wave model: one resident wave costs the measured 72.3 us
    assert abs(plan["predicted_slice_time"] - 72_320) < 5_000 or plan["blocks_per_slice"] < 147
