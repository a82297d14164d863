"""Live B200 runs of the BASELINE configs through the C++ scheduler (include/ms_live.h).

Python only allocates the tenants' synthetic tensors, registers the sm_100a kernels,
and hands the scenario + bindings to ms_live_run, which runs Algorithm 1 in C++ on
this thread in real time.  Policies: splitkernel (this system), exclusive (HP alone ->
SLO), exclusive_lp (LP alone -> LP throughput reference), reef / reef_req
(kernel-boundary temporal sharing baselines).
"""
from __future__ import annotations

import ctypes as C
import json
import math
import time

from . import scenarios
from .device import Device, _ck, lib as dev_lib

SEED = 20260117
DEFAULT_LP_SM_RESERVE = int(__import__("os").environ.get("MS_LP_SM_RESERVE", "1"))  # ms_b200.cu ms_dev::lp_sm_reserve (the HP gate's home)


def _live_lib():
    L = dev_lib()
    if not hasattr(L, "_ms_live_sig"):
        L.ms_live_run.restype = C.c_int
        L.ms_live_run.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                  C.POINTER(C.c_void_p)]
        L.ms_live_free.argtypes = [C.c_void_p]
        L._ms_live_sig = True
    return L


def live_run(dev: Device, scenario: dict, policy: str, binding: dict, options: dict | None = None) -> dict:
    L = _live_lib()
    out = C.c_void_p()
    rc = L.ms_live_run(dev._h, json.dumps(scenario).encode(), policy.encode(), json.dumps(binding).encode(),
                       json.dumps(options or {}).encode(), C.byref(out))
    if rc != 0:
        raise RuntimeError(f"ms_live_run({policy}) failed rc={rc}: {L.ms_last_error().decode(errors='replace')}")
    s = C.cast(out, C.c_char_p).value.decode()
    L.ms_live_free(out)
    return json.loads(s)


class Config1:
    """Config 1 tenants on one B200: HP = 4 x (C[128x4096] = A[128x4096] W_i^T) + bias/GELU,
    LP = bf16 GEMM loop M = N = K = 8192 (128x256 tiles, 2048 tiles per GEMM)."""

    M_HP, H = 128, 4096
    N_LP = 8192

    def __init__(self, dev: Device, seed: int = SEED):
        self.dev = dev
        n, H, M = self.N_LP, self.H, self.M_HP
        self.a = dev.alloc(n * n * 2)
        self.b = dev.alloc(n * n * 2)
        self.c = dev.alloc(n * n * 2)
        dev.fill_synth(self.a, n * n, seed, 1, 1.0)
        dev.fill_synth(self.b, n * n, seed, 2, 1.0 / math.sqrt(n))
        self.lp = dev.lp_register_gemm(self.a, self.b, self.c, n, n, n, block_n=256)
        self.act = [dev.alloc(M * H * 2) for _ in range(5)]
        self.w = [dev.alloc(H * H * 2) for _ in range(4)]
        self.bias = dev.alloc(H * 2)
        dev.fill_synth(self.act[0], M * H, seed, 100, 1.0)
        for i, w in enumerate(self.w):
            dev.fill_synth(w, H * H, seed, 101 + i, 1.0 / math.sqrt(H))
        dev.fill_synth(self.bias, H, seed, 110, 0.1)
        ops = [dict(kind=1, block_n=128, a=self.act[i], b=self.w[i], c=self.act[i + 1], bias=0, m=M, n=H, k=H)
               for i in range(4)]
        ops.append(dict(kind=2, block_n=0, a=self.act[4], b=0, c=self.act[0], bias=self.bias, m=M, n=H, k=0))
        self.chain = dev.hp_register_chain(ops)
        # e2e chain: the request's input activation arrives from pinned host memory after
        # the doorbell and the output returns to pinned host memory before completion.
        self.io_bytes = M * H * 2
        self.host_in = dev.host_alloc(self.io_bytes)
        self.host_out = dev.host_alloc(self.io_bytes)
        self.act_out = dev.alloc(self.io_bytes)
        dev.d2h(self.host_in, self.act[0], self.io_bytes)
        e2e = [dict(kind=3, block_n=0, a=self.host_in, b=0, c=self.act[0], bias=0, m=self.io_bytes, n=0, k=0)]
        e2e += ops[:4]
        e2e.append(dict(kind=2, block_n=0, a=self.act[4], b=0, c=self.act_out, bias=self.bias, m=M, n=H, k=0))
        e2e.append(dict(kind=4, block_n=0, a=self.act_out, b=0, c=self.host_out, bias=0, m=self.io_bytes, n=0, k=0))
        self.chain_e2e = dev.hp_register_chain(e2e)
        self.calib = None

    def binding(self, e2e: bool = False) -> dict:
        return {"lp": {"lp_gemm_8192": self.lp.id}, "hp": {"hp_infer": [self.chain_e2e if e2e else self.chain]}}

    def calibrate(self, reps: int = 5, profile: bool = True) -> dict:
        """Measured per-tile / per-chain times feeding both the live pacing and the replay
        scenario (KernelSpec calibrated from the B200 kernels).  `profile`:
        also the on-B200 profile of the LP GEMM over tile prefixes (profiler.py), which the
        scenario carries as KernelSpec.measured_time — the reference's measured execution
        oracle for split plans (engine.hpp:461-481, splitter.hpp:141-207)."""
        self.dev.set_lp_sm_reserve(DEFAULT_LP_SM_RESERVE)  # a live run may have left a governed reserve
        ms_gemm = self.dev.lp_time_full(self.lp, reps)
        waves = math.ceil(self.lp.total_tiles / (self.dev.info["sm_count"] // self.lp.tile_ctas))
        ms_chain = self.dev.hp_time_chain(self.chain, 20)
        tile_ns = int(ms_gemm * 1e6 / waves)
        self.calib = {
            "lp_gemm_ms": ms_gemm,
            "lp_gemm_tile_ns": tile_ns,
            "lp_gemm_tiles": int(self.lp.total_tiles),
            "lp_gemm_tile_ctas": int(self.lp.tile_ctas),
            "hp_chain_ms": ms_chain,
            "hp_gemm_tile_ns": int(ms_chain * 1e6 * 0.95 / 4),
            "hp_ew_tile_ns": max(1000, int(ms_chain * 1e6 * 0.05)),
        }
        if profile:
            from . import profiler
            sm = self.dev.info["sm_count"]
            spec = profiler.profile_lp_kernel(self.dev, self.lp, "lp_gemm_8192", sm // self.lp.tile_ctas,
                                              scenarios.DEFAULT_CALIB["lp_gemm_tile_bytes"], reps=2)
            self.calib["lp_gemm_measured_time"] = spec["measured_time"]
        return self.calib

    def scenario(self, seed: int, horizon_s: float) -> dict:
        return scenarios.config1(seed=seed, horizon_s=horizon_s, calib=self.calib or {})

    def options(self, **kw) -> dict:
        o = {"tile_ns": {"lp_gemm_8192": (self.calib or {}).get("lp_gemm_tile_ns", 57000)}, "timeline": True}
        o.update(kw)
        return o


def decode_step_ops(M: int, H: int, Q: int, F: int, V: int, layers: int, bufs, weights, lm) -> list[dict]:
    """HP chain of one synthetic Llama-style decode step (config 4): per layer
    qkv = h Wqkv^T, o = qkv[:, :H] Wo^T (strided A: the attention core is not modelled),
    act = silu(o Wg^T) * (o Wu^T) (one GEMM_SWIGLU op, Wgu = [Wg; Wu]), h = act Wd^T; then
    logits = h Wlm^T.  `bufs` = (h, qkv, o, gu, act, logits) device pointers (gu unused by
    the fused SwiGLU); `weights[l]` = (Wqkv, Wo, Wgu, Wd)."""
    h, qkv, o, gu, act, logits = bufs
    ops = []
    for l in range(layers):
        wq, wo, wg, wd = weights[l]
        ops += [dict(kind=1, block_n=128, a=h, b=wq, c=qkv, bias=0, m=M, n=Q, k=H),
                dict(kind=1, block_n=128, a=qkv, b=wo, c=o, bias=0, m=M, n=H, k=H, lda=Q),
                dict(kind=6, block_n=128, a=o, b=wg, c=act, bias=0, m=M, n=F, k=H),
                dict(kind=1, block_n=128, a=act, b=wd, c=h, bias=0, m=M, n=H, k=F)]
    ops.append(dict(kind=1, block_n=128, a=h, b=lm, c=logits, bias=0, m=M, n=V, k=H))
    return ops


class Config4:
    """Config 4 tenants on one B200.  HP = one bs=1 decode step of a Llama-3.2-1B-geometry
    model (hidden 2048, qkv 3072, FFN 8192, 16 layers, vocab 128256: 1.24 B parameters =
    2.47 GB of bf16 weights streamed per token) as an m = 1 chain, i.e. the HBM-streaming
    GEMV chain (hp_gemv.cuh).  LP1 = bf16 8192^3 GEMM loop, LP2 = bf16 axpy over 2^30
    elements (6 GiB of HBM traffic per pass).  m = 128 gives the tcgen05 chain with the token
    in row 0 of the UMMA tile (round-1 layout, kept for comparison)."""

    M, H, Q, F, V, LAYERS = 1, 2048, 3072, 8192, 128256, 16
    N_LP = 8192
    N_EW = 1 << 30

    def __init__(self, dev: Device, seed: int = SEED, m: int | None = None, tier=None, slow_max: int = 8,
                 lp_split: int = 1):
        """tier: a MemoryTier (tier.py) to place the tenants' memory through — HP buffers
        and weights pinned (task 0), LP GEMM (task 1) and streamer (task 2) spillable, in
        that allocation order (the memory-intensive case)."""
        self.dev = dev
        if m is not None:
            self.M = m
        hp_alloc = (lambda nb: tier.alloc(0, nb, high_priority=True)) if tier else dev.alloc
        gemm_alloc = (lambda nb: tier.alloc(1, nb)) if tier else dev.alloc
        ew_alloc = (lambda nb: tier.alloc(2, nb)) if tier else dev.alloc
        M, H, Q, F, V = self.M, self.H, self.Q, self.F, self.V
        self.bufs = [hp_alloc(M * n * 2) for n in (H, Q, H, 2 * F, F, V)]
        dev.fill_synth(self.bufs[0], M * H, seed, 400, 1.0)
        self.weights = []
        for l in range(self.LAYERS):
            ws = []
            for j, (n, k) in enumerate([(Q, H), (H, H), (2 * F, H), (H, F)]):
                p = hp_alloc(n * k * 2)
                dev.fill_synth(p, n * k, seed, 401 + 4 * l + j, 1.0 / math.sqrt(k))
                ws.append(p)
            self.weights.append(ws)
        self.lm = hp_alloc(V * H * 2)
        dev.fill_synth(self.lm, V * H, seed, 499, 1.0 / math.sqrt(H))
        self.chain = dev.hp_register_chain(decode_step_ops(M, H, Q, F, V, self.LAYERS, self.bufs,
                                                           self.weights, self.lm))
        n = self.N_LP
        self.a, self.b, self.c = gemm_alloc(n * n * 2), gemm_alloc(n * n * 2), gemm_alloc(n * n * 2)
        dev.fill_synth(self.a, n * n, seed, 1, 1.0)
        dev.fill_synth(self.b, n * n, seed, 2, 1.0 / math.sqrt(n))
        # lp_split > 1: 128 x 256 tiles cut into k-slices (shorter preemption grain, finer
        # harvest packing; fp32 partials reduced in-kernel)
        self.lp_gemm = dev.lp_register_gemm(self.a, self.b, self.c, n, n, n, block_n=256, split_k=lp_split)
        self.x, self.y = ew_alloc(self.N_EW * 2), ew_alloc(self.N_EW * 2)
        dev.fill_synth(self.x, self.N_EW, seed, 21, 1.0)
        dev.fill_synth(self.y, self.N_EW, seed, 22, 1.0)
        # 8192-element tiles (7.0 TB/s).  4096 cut the preemption drain from ~11 to ~8 us and the
        # config-4 ring -> first HP CTA p99 from ~10.3 to ~6.5 us, but the governor then granted
        # LP ~90 instead of ~78 SMs and HP SLO attainment fell 4-9 points below exclusive in
        # three runs (tools/axpy_probe.py, tools/policy_compare.py)
        self.lp_axpy = dev.lp_register_axpy(self.x, self.y, self.N_EW, 0.5, tile_elems=8192)
        if tier is not None and slow_max:
            slow = tier.off_device(self.x, self.y)
            if any(slow):  # bound the drain over PCIe / NVLink (ms_lp_set_slow_tiles)
                dev.lp_set_slow_tiles(self.lp_axpy, slow, tier.CHUNK // (2 * 8192), slow_max)
        self.calib = None

    @property
    def weight_bytes(self) -> int:
        H, Q, F, V = self.H, self.Q, self.F, self.V
        return 2 * (self.LAYERS * (Q * H + H * H + 2 * F * H + H * F) + V * H)

    def binding(self) -> dict:
        return {"lp": {"lp_gemm_8192": self.lp_gemm.id, "lp_axpy_1g": self.lp_axpy.id},
                "hp": {"hp_decode": [self.chain]}}

    def calibrate(self, reps: int = 3) -> dict:
        self.dev.set_lp_sm_reserve(DEFAULT_LP_SM_RESERVE)
        sm = self.dev.info["sm_count"]
        ms_gemm = self.dev.lp_time_full(self.lp_gemm, reps)
        ms_axpy = self.dev.lp_time_full(self.lp_axpy, reps)
        # HP step alone, after the LP timing runs: the part leaves its power cap within
        # ~0.1 s; take the best of three (the request rate is derived from this number)
        time.sleep(0.3)
        ms_chain = min(self.dev.hp_time_chain(self.chain, 5) for _ in range(3))
        self.calib = {
            "lp_gemm_ms": ms_gemm, "lp_axpy_ms": ms_axpy, "hp_step_ms": ms_chain,
            "hp_weight_gbs": self.weight_bytes / (ms_chain * 1e-3) / 1e9,
            "lp_gemm_tile_ns": int(ms_gemm * 1e6 / math.ceil(self.lp_gemm.total_tiles / (sm // self.lp_gemm.tile_ctas))),
            "lp_gemm_tiles": int(self.lp_gemm.total_tiles),
            "lp_gemm_tile_ctas": int(self.lp_gemm.tile_ctas),
            # one "tile" of the pacing model = one tile per SM per wave
            "lp_ew_tile_ns": int(ms_axpy * 1e6 / math.ceil(self.lp_axpy.total_tiles / sm)),
            "lp_ew_tiles": int(self.lp_axpy.total_tiles),
            "lp_ew_tile_bytes": 6 * 8192,
            "hp_layer_ns": int(ms_chain * 1e6 * 0.79 / self.LAYERS),
            "hp_lm_head_ns": int(ms_chain * 1e6 * 0.21),
        }
        # on-B200 profiles -> KernelSpec.measured_time of both LP kernels (profiler.py)
        from . import profiler
        self.calib["lp_gemm_measured_time"] = profiler.profile_lp_kernel(
            self.dev, self.lp_gemm, "lp_gemm_8192", sm // self.lp_gemm.tile_ctas, scenarios.DEFAULT_CALIB["lp_gemm_tile_bytes"],
            reps=1)["measured_time"]
        self.calib["lp_ew_measured_time"] = profiler.profile_lp_kernel(
            self.dev, self.lp_axpy, "lp_axpy_1g", 3 * (sm - 1), 6 * 8192, reps=1)["measured_time"]
        return self.calib

    def hp_rate(self, utilisation: float = 0.5) -> float:
        """Request rate giving the HP tenant `utilisation` of the GPU on its own.  At the
        specified 20 req/s the HP tenant alone is overloaded on B200 (2.47 GB of weights per
        token, 80 tokens per request on average, plus 0.3 ms of CPU gap per token)."""
        step_s = (self.calib or {}).get("hp_step_ms", 1.0) * 1e-3
        return utilisation / (80.0 * (step_s + 300e-6))

    # Large-bubble threshold for the live runs (the reference's scheduler.threshold_ms,
    # default 2 ms): with µs-scale preemption there is no reason to leave a gap between
    # decode requests idle for 2 ms before harvesting it (the request-level kernel-boundary
    # baseline relaunches LP the moment HP has no request); as for configs 2/3.
    THRESHOLD_MS = 0.02

    def scenario(self, seed: int, horizon_s: float, rate: float | None = None) -> dict:
        return scenarios.config4(seed=seed, horizon_s=horizon_s, calib=self.calib or {},
                                 rate=rate if rate is not None else self.hp_rate(), threshold_ms=self.THRESHOLD_MS)

    def options(self, **kw) -> dict:
        c = self.calib or {}
        o = {"tile_ns": {"lp_gemm_8192": c.get("lp_gemm_tile_ns", 57000),
                         "lp_axpy_1g": c.get("lp_ew_tile_ns", 4000)}, "timeline": True}
        o.update(kw)
        return o


class _TrainInferConfig:
    """Shared shape of configs 2 and 3: one HP inference tenant (a per-op chain of one
    request, 1 iteration, Poisson arrivals) + one LP training-step tenant (TrainStepLP)."""

    HP_TASK = LP_TASK = NAME = ""
    RATE = 100.0
    # Large-bubble threshold (the reference's scheduler.threshold_ms, default 2 ms): these HP
    # tenants have no in-request hints, so LP runs only between requests; with a preemption
    # that costs a few us there is no reason to let a gap of a few ms idle for 2 ms first.
    THRESHOLD_MS = 0.02

    def _finish(self, dev: Device, hp, lp):
        self.dev, self.hp, self.lp = dev, hp, lp
        self.chain = dev.hp_register_chain(hp.ops)
        self.calib = None

    def calibrate(self, reps: int = 2) -> dict:
        c = self.lp.calibrate(reps)
        time.sleep(0.2)
        ms_chain = min(self.dev.hp_time_chain(self.chain, 10) for _ in range(3))
        self.calib = dict(c, hp_chain_ms=ms_chain, hp_gemm_tflops=self.hp.gemm_flops / (ms_chain * 1e-3) / 1e12,
                          hp_ops=len(self.hp.ops), lp_tile_ns=dict(self.lp.tile_ns))
        return self.calib

    def hp_rate(self, max_util: float = 0.8) -> float:
        """The config's request rate, capped so HP alone stays <= max_util."""
        ms = (self.calib or {}).get("hp_chain_ms", 1.0)
        return min(self.RATE, max_util / (ms * 1e-3))

    def scenario(self, seed: int, horizon_s: float, rate: float | None = None) -> dict:
        c = self.calib or {}
        return scenarios.train_infer(self.NAME, seed=seed, horizon_s=horizon_s, hp_task=self.HP_TASK,
                                     hp_ops=len(self.hp.ops), hp_chain_ns=int(c.get("hp_chain_ms", 1.0) * 1e6),
                                     lp_task=self.LP_TASK, lp_specs=self.lp.kernel_specs(),
                                     lp_sequence=self.lp.sequence, rate=rate or self.hp_rate(),
                                     threshold_ms=self.THRESHOLD_MS)

    def binding(self) -> dict:
        return {"lp": self.lp.binding(), "hp": {self.HP_TASK: [self.chain]}}

    def options(self, **kw) -> dict:
        o = {"tile_ns": dict(self.lp.tile_ns), "timeline": True}
        o.update(kw)
        return o

    def close(self):
        self.dev.hp_unregister_chain(self.chain)
        self.hp.free()
        self.lp.free()


class Config2(_TrainInferConfig):
    """Config 2 (BASELINE configs[1]): HP ResNet-50 bs=1 inference (76-op chain: im2col +
    tcgen05 conv GEMMs with folded-BN / residual / ReLU epilogues + pools + FC) at 200 req/s,
    LP ResNet-50 training step at bs=64 (48 distinct conv/FC GEMM shapes fwd/dgrad/wgrad +
    SGD)."""

    HP_TASK, LP_TASK, NAME, RATE = "hp_resnet50", "lp_resnet50_train", "cfg2_resnet50", 200.0

    def __init__(self, dev: Device, seed: int = SEED):
        from .tenants import RESNET50_PARAMS, ResNet50HP, TrainStepLP, resnet50_train_gemms
        hp = ResNet50HP(dev, seed)
        lp = TrainStepLP(dev, "rn50", resnet50_train_gemms(64), RESNET50_PARAMS, optim_mode=1, seed=seed,
                         tensor_base=2900)
        self._finish(dev, hp, lp)


class Config3(_TrainInferConfig):
    """Config 3 (BASELINE configs[2]): HP BERT-base bs=1 seq-128 encoder (84-op chain) at
    100 req/s, LP BERT-base training step at bs=32 (9 distinct GEMM shapes x 144 GEMMs +
    AdamW over 110 M parameters)."""

    HP_TASK, LP_TASK, NAME, RATE = "hp_bert", "lp_bert_train", "cfg3_bert_base", 100.0

    def __init__(self, dev: Device, seed: int = SEED):
        from .tenants import BERT_PARAMS, BertHP, TrainStepLP, bert_train_gemms
        hp = BertHP(dev, seed)
        lp = TrainStepLP(dev, "bert", bert_train_gemms(32), BERT_PARAMS, optim_mode=0, seed=seed, tensor_base=3900)
        self._finish(dev, hp, lp)
