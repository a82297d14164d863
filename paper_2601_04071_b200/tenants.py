"""Tenant workloads of BASELINE.json configs[1] and configs[2]:

  config 2: HP ResNet-50 bs=1 224x224 inference (53 convolutions as tcgen05 GEMMs over
            im2col patch matrices with the folded-BN bias + residual + ReLU fused in the GEMM
            epilogue, 3x3/2 max pool, global average pool, FC 2048 -> 1000) + LP ResNet-50
            training step at
            bs=64 (the fwd / dgrad / wgrad GEMM of every convolution and the FC at their
            true shapes, then an SGD-momentum step over the 25.6 M parameters);
  config 3: HP BERT-base bs=1 seq 128 encoder (12 x {QKV GEMM, attention, O GEMM,
            residual + LayerNorm, FFN1 GEMM with bias/GELU epilogue, FFN2 GEMM, residual +
            LayerNorm})
            + LP BERT-base training step at bs=32 seq 128 (the 12 GEMMs of each of the 12
            layers, fwd + dgrad + wgrad, then AdamW over 110 M parameters).

Everything is synthetic (no checkpoints / datasets): weights U[-1, 1) * sqrt(6 / fan_in)
(He-uniform), biases U[-0.1, 0.1), input U[-1, 1), keyed by (seed, tensor id) with the
generator shared with oracle/tenant_ref.c.  Activations are NHWC, batch 1, rows padded to
the 128-row GEMM tile (pad rows are computed and never read as data).

This module only lays out buffers and op lists; every op runs in the sm_100a kernels behind
include/ms_b200.h (tcgen05 GEMM tc_gemm.cuh, glue ops hp_ops.cuh, optimizer lp_optim.cuh).
The LP training steps keep the GEMMs' shapes, order and FLOPs but not the data flow
between them: each GEMM reads / writes shared scratch operands (a scheduler tenant, not a
trainer), stated in DESIGN.md §3.
"""
from __future__ import annotations

import math

from .device import MS_HP_ADD_LN, MS_HP_ATTN, MS_HP_AVGPOOL, MS_HP_GEMM, MS_HP_IM2COL, MS_HP_MAXPOOL, Device


def pad_to(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def block_n_for(n: int) -> int:
    return 256 if n % 256 == 0 else 128 if n % 128 == 0 else 64


# ----------------------------------------------------------------------------- ResNet-50
RESNET50_STAGES = ((64, 256, 3, 1), (128, 512, 4, 2), (256, 1024, 6, 2), (512, 2048, 3, 2))


def resnet50_convs() -> list[dict]:
    """The 53 convolutions of ResNet-50 (v1.5: stride on the 3x3), in forward order, plus
    the FC as a 1x1 'conv' over the pooled vector."""
    convs = [dict(name="conv1", cin=3, cout=64, k=7, s=2, p=3, hin=224, relu=True, role="stem")]
    h, cin = 56, 64
    for si, (mid, out, n, stride) in enumerate(RESNET50_STAGES):
        for b in range(n):
            s = stride if b == 0 else 1
            tag = f"s{si + 1}b{b + 1}"
            convs.append(dict(name=f"{tag}_reduce", cin=cin, cout=mid, k=1, s=1, p=0, hin=h, relu=True, role="reduce"))
            convs.append(dict(name=f"{tag}_conv3", cin=mid, cout=mid, k=3, s=s, p=1, hin=h, relu=True, role="conv3"))
            convs.append(dict(name=f"{tag}_expand", cin=mid, cout=out, k=1, s=1, p=0, hin=h // s, relu=True,
                              role="expand"))
            if b == 0:
                convs.append(dict(name=f"{tag}_down", cin=cin, cout=out, k=1, s=s, p=0, hin=h, relu=False,
                                  role="down"))
            h, cin = h // s, out
    return convs


def conv_out(c: dict) -> int:
    return (c["hin"] + 2 * c["p"] - c["k"]) // c["s"] + 1


class ResNet50HP:
    """HP tenant of config 2: one bs=1 224x224 inference as one HP chain (per-op kernels,
    PDL-linked, pre-armed behind the doorbell gate).  `ops` is the ms_hp_op list; `bufs`
    maps buffer name -> (device pointer, bytes) for the oracle chain check."""

    N_CLASSES, FC_PAD = 1000, 1024

    def __init__(self, dev: Device, seed: int, tensor_base: int = 2000):
        self.dev, self.seed = dev, seed
        self.bufs: dict[str, tuple[int, int]] = {}
        self.ops: list[dict] = []
        self.weights: dict[str, tuple] = {}  # name -> (ptr, rows, cols, tensor id, scale)
        tid = [tensor_base]

        def buf(name, rows, cols):
            nb = rows * cols * 2
            p = dev.alloc(nb)
            dev.memset(p, 0, nb)
            self.bufs[name] = (p, nb)
            return p

        def weight(name, rows, cols, scale):
            p = dev.alloc(rows * cols * 2)
            tid[0] += 1
            dev.fill_synth(p, rows * cols, seed, tid[0], scale)
            self.weights[name] = (p, rows, cols, tid[0], scale)
            self.bufs[name] = (p, rows * cols * 2)
            return p

        def gemm(a, w, c, m, n, k, bias=0, resid=0, relu=False):
            """tcgen05 GEMM op with the conv epilogue fused (folded-BN shift, residual, ReLU on
            the fp32 accumulators: ms_hp_op.bias / resid / geo.flags)."""
            self.ops.append(dict(kind=MS_HP_GEMM, block_n=block_n_for(n), a=a, b=w, c=c, bias=bias, m=m, n=n, k=k,
                                 resid=resid, geo=dict(flags=1 if relu else 0)))

        def conv(c, x, name, resid=0):
            """conv c (+ bias, + resid, ReLU per c["relu"]) over NHWC x ([pad(hin^2) x cin])."""
            ho = conv_out(c)
            m = pad_to(ho * ho, 128)
            kvalid = c["k"] * c["k"] * c["cin"]
            kp = pad_to(kvalid, 64)
            if c["k"] == 1 and c["s"] == 1:
                a = x
            else:
                a = buf(f"{name}.col", m, kp)
                self.ops.append(dict(kind=MS_HP_IM2COL, block_n=0, a=x, b=0, c=a, bias=0, m=m, n=kp, k=0,
                                     geo=dict(h=c["hin"], w=c["hin"], cin=c["cin"], kh=c["k"], kw=c["k"], stride=c["s"],
                                              pad=c["p"])))
            w = weight(f"{name}.w", c["cout"], kp, math.sqrt(6.0 / kvalid))
            bias = weight(f"{name}.b", 1, c["cout"], 0.1)
            y = buf(f"{name}.out", m, c["cout"])
            gemm(a, w, y, m, c["cout"], kp, bias=bias, resid=resid, relu=c["relu"])
            return y, m

        # stem
        self.input = buf("input", 224 * 224, 3)
        tid[0] += 1
        self.input_tensor = tid[0]
        dev.fill_synth(self.input, 224 * 224 * 3, seed, self.input_tensor, 1.0)
        convs = resnet50_convs()
        x, m = conv(convs[0], self.input, "conv1")
        mp = buf("pool1", pad_to(56 * 56, 128), 64)
        self.ops.append(dict(kind=MS_HP_MAXPOOL, block_n=0, a=x, b=0, c=mp, bias=0, m=pad_to(56 * 56, 128), n=64, k=0,
                             geo=dict(h=112, w=112, cin=64, kh=3, kw=3, stride=2, pad=1)))
        x = mp
        i = 1
        while i < len(convs):
            red, c3, ex = convs[i], convs[i + 1], convs[i + 2]
            down = convs[i + 3] if i + 3 < len(convs) and convs[i + 3]["role"] == "down" else None
            t1, _ = conv(red, x, red["name"])
            t2, _ = conv(c3, t1, c3["name"])
            resid = x
            if down:  # projection shortcut first: the expand conv's epilogue adds it
                resid, _ = conv(down, x, down["name"])
            x, _ = conv(ex, t2, ex["name"], resid=resid)
            i += 4 if down else 3
        # head: global average pool (row 0) -> FC (1000 classes padded to 1024) -> + bias
        pooled = buf("avgpool", 128, 2048)
        self.ops.append(dict(kind=MS_HP_AVGPOOL, block_n=0, a=x, b=0, c=pooled, bias=0, m=128, n=2048, k=0,
                             geo=dict(h=7, w=7)))
        wfc = weight("fc.w", self.FC_PAD, 2048, math.sqrt(6.0 / 2048))
        bfc = weight("fc.b", 1, self.FC_PAD, 0.1)
        self.logits = buf("logits", 128, self.FC_PAD)
        gemm(pooled, wfc, self.logits, 128, self.FC_PAD, 2048, bias=bfc)

    @property
    def gemm_flops(self) -> int:
        return sum(2 * o["m"] * o["n"] * o["k"] for o in self.ops if o["kind"] == MS_HP_GEMM)

    def free(self):
        for p, _ in self.bufs.values():
            self.dev.free(p)
        self.bufs.clear()


def resnet50_train_gemms(batch: int = 64) -> list[tuple[str, int, int, int]]:
    """The GEMMs of one ResNet-50 training step at `batch`, in execution order: forward
    (conv i: M = batch*Ho*Wo, N = Cout, K = Cin*k*k), then backward in reverse layer order
    (dgrad: M = batch*Ho*Wo, N = Cin*k*k, K = Cout — skipped for the stem; wgrad: M = Cout,
    N = Cin*k*k, K = batch*Ho*Wo), FC included.  Shapes padded to the tile (M 128, N 64,
    K 64).  Returns (role, m, n, k)."""
    convs = resnet50_convs() + [dict(name="fc", cin=2048, cout=1000, k=1, s=1, p=0, hin=1, relu=False, role="fc")]
    fwd, bwd = [], []
    for c in convs:
        ho = conv_out(c)
        mrows = batch * ho * ho
        kk = c["cin"] * c["k"] * c["k"]
        fwd.append(("fwd", pad_to(mrows, 128), pad_to(c["cout"], 64), pad_to(kk, 64)))
        g = []
        if c["role"] != "stem":
            g.append(("dgrad", pad_to(mrows, 128), pad_to(kk, 64), pad_to(c["cout"], 64)))
        g.append(("wgrad", pad_to(c["cout"], 128), pad_to(kk, 64), pad_to(mrows, 64)))
        bwd.append(g)
    out = list(fwd)
    for g in reversed(bwd):
        out += g
    return out


RESNET50_PARAMS = 25_557_032


# ----------------------------------------------------------------------------- BERT-base
BERT = dict(hidden=768, heads=12, ffn=3072, layers=12, seq=128)


class BertHP:
    """HP tenant of config 3: one BERT-base encoder pass (bs=1, seq 128) as one HP chain."""

    def __init__(self, dev: Device, seed: int, tensor_base: int = 3000, layers: int | None = None):
        self.dev, self.seed = dev, seed
        S, D, F = BERT["seq"], BERT["hidden"], BERT["ffn"]
        L = layers or BERT["layers"]
        self.bufs: dict[str, tuple[int, int]] = {}
        self.ops: list[dict] = []
        self.weights: dict[str, tuple] = {}
        tid = [tensor_base]

        def buf(name, rows, cols):
            nb = rows * cols * 2
            p = dev.alloc(nb)
            dev.memset(p, 0, nb)
            self.bufs[name] = (p, nb)
            return p

        def weight(name, rows, cols, scale):
            p = dev.alloc(rows * cols * 2)
            tid[0] += 1
            dev.fill_synth(p, rows * cols, seed, tid[0], scale)
            self.weights[name] = (p, rows, cols, tid[0], scale)
            self.bufs[name] = (p, rows * cols * 2)
            return p

        def gemm(a, w, c, n, k):
            self.ops.append(dict(kind=MS_HP_GEMM, block_n=128, a=a, b=w, c=c, bias=0, m=S, n=n, k=k))

        self.input = buf("input", S, D)
        tid[0] += 1
        self.input_tensor = tid[0]
        dev.fill_synth(self.input, S * D, seed, self.input_tensor, 1.0)
        x = self.input
        for l in range(L):
            t = f"l{l}"
            qkv = buf(f"{t}.qkv", S, 3 * D)
            gemm(x, weight(f"{t}.wqkv", 3 * D, D, math.sqrt(6.0 / D)), qkv, 3 * D, D)
            ctx = buf(f"{t}.ctx", S, D)
            self.ops.append(dict(kind=MS_HP_ATTN, block_n=0, a=qkv, b=0, c=ctx, bias=0, m=S, n=D, k=0))
            o = buf(f"{t}.o", S, D)
            gemm(ctx, weight(f"{t}.wo", D, D, math.sqrt(6.0 / D)), o, D, D)
            x1 = buf(f"{t}.x1", S, D)
            self.ops.append(dict(kind=MS_HP_ADD_LN, block_n=0, a=o, b=x, c=x1, bias=weight(f"{t}.ln1", 2, D, 1.0),
                                 m=S, n=D, k=0))
            g = buf(f"{t}.ffn1_gelu", S, F)  # FFN1 + bias + GELU fused in the GEMM epilogue
            self.ops.append(dict(kind=MS_HP_GEMM, block_n=128, a=x1, b=weight(f"{t}.w1", F, D, math.sqrt(6.0 / D)),
                                 c=g, bias=weight(f"{t}.b1", 1, F, 0.1), m=S, n=F, k=D, geo=dict(flags=2)))
            f2 = buf(f"{t}.ffn2", S, D)
            gemm(g, weight(f"{t}.w2", D, F, math.sqrt(6.0 / F)), f2, D, F)
            x2 = buf(f"{t}.out", S, D)
            self.ops.append(dict(kind=MS_HP_ADD_LN, block_n=0, a=f2, b=x1, c=x2, bias=weight(f"{t}.ln2", 2, D, 1.0),
                                 m=S, n=D, k=0))
            x = x2
        self.output = x

    @property
    def gemm_flops(self) -> int:
        return sum(2 * o["m"] * o["n"] * o["k"] for o in self.ops if o["kind"] == MS_HP_GEMM)

    def free(self):
        for p, _ in self.bufs.values():
            self.dev.free(p)
        self.bufs.clear()


def bert_train_gemms(batch: int = 32) -> list[tuple[str, int, int, int]]:
    """GEMMs of one BERT-base training step (bs x seq tokens): per layer fwd QKV, O, FFN1,
    FFN2; backward in reverse (dgrad then wgrad per linear).  (role, m, n, k)."""
    T, D, F, L = batch * BERT["seq"], BERT["hidden"], BERT["ffn"], BERT["layers"]
    lin = [(3 * D, D), (D, D), (F, D), (D, F)]  # (out, in) of QKV, O, FFN1, FFN2
    out = []
    for _ in range(L):
        out += [("fwd", T, n, k) for n, k in lin]
    for _ in range(L):
        for n, k in reversed(lin):
            out += [("dgrad", T, k, n), ("wgrad", n, k, T)]
    return out


BERT_PARAMS = 109_482_240


# ----------------------------------------------------------------------------- LP training step
def step_plan(prefix: str, gemms: list[tuple[str, int, int, int]], optim_mode: int):
    """Distinct GEMM shapes of a training step -> kernel names, and the step's kernel order
    as (name, repeat) runs ending with the optimizer.  Pure (no device): the scenario
    builder and the CPU replay tests use it too."""
    shapes: dict[tuple[int, int, int], str] = {}
    sequence: list[tuple[str, int]] = []
    for _, m, n, k in gemms:
        nm = shapes.setdefault((m, n, k), f"{prefix}_g{m}x{n}x{k}")
        if sequence and sequence[-1][0] == nm:
            sequence[-1] = (nm, sequence[-1][1] + 1)
        else:
            sequence.append((nm, 1))
    optim_name = f"{prefix}_{'adamw' if optim_mode == 0 else 'sgd'}"
    sequence.append((optim_name, 1))
    return {nm: shp for shp, nm in shapes.items()}, sequence, optim_name


def kernel_spec(name: str, tiles: int, tile_ns: int, tile_bytes: int, per_sm: int = 1, measured_time=None) -> dict:
    """Reference-schema KernelSpec (scenario_io.hpp) of a persistent preemptible LP kernel:
    grid = tile count, one CTA per SM (tpb 256, occupancy per_sm/8 -> Eq. 1 = 148 * per_sm),
    block_time = per-wave tile time, bandwidth = the tile's compulsory bytes / tile time."""
    k = {"name": name, "grid": [int(tiles), 1, 1], "threads_per_block": 256, "occupancy": per_sm / 8.0,
         "block_time": {"dist": "point", "value": {"value": int(tile_ns), "unit": "ns"}},
         "bw_demand_per_block": float(tile_bytes) / (tile_ns * 1e-9), "splittable": True}
    if measured_time:  # on-B200 profile rows -> the reference's measured oracle (engine.hpp:461-481)
        k["measured_time"] = measured_time
    return k


def gemm_tiles(m: int, n: int) -> int:
    return (m // 128) * (n // block_n_for(n))


def split_for(m: int, n: int, k: int, sms: int = 147, max_unit_kb: int = 64, min_unit_kb: int = 8) -> int:
    """k-slices per tile of an LP training GEMM: enough units to fill the GPU when the GEMM
    has few tiles and a long K (the wgrad GEMMs reduce over the whole batch: K up to 802,816),
    and no unit longer than `max_unit_kb` k-blocks (the preemption grain: 128 x 256 x 4096
    bf16 is ~30 us on one SM).  A power of two dividing K / 64."""
    kb, tiles = k // 64, gemm_tiles(m, n)
    split = 1
    while kb % (2 * split) == 0 and kb // (2 * split) >= min_unit_kb and (
            tiles * split < sms or kb // split > max_unit_kb):
        split *= 2
    return split


def gemm_tile_bytes(n: int, k: int) -> int:
    bn = block_n_for(n)
    return (128 + bn) * k * 2 + 128 * bn * 2


def step_specs(prefix: str, gemms, n_params: int, optim_mode: int, tile_ns: dict | None = None,
               measured: dict | None = None) -> tuple:
    """(specs, sequence) of a training step without a device (tile times default to a
    roofline estimate at 1300 TFLOP/s / 6.5 TB/s over 147 SMs)."""
    shapes, sequence, optim_name = step_plan(prefix, gemms, optim_mode)
    tile_ns, measured = tile_ns or {}, measured or {}
    specs = []
    for nm, (m, n, k) in shapes.items():
        sp = split_for(m, n, k)
        est = int(2 * 128 * block_n_for(n) * (k // sp) / (1300e12 / 147) * 1e9)
        specs.append(kernel_spec(nm, gemm_tiles(m, n) * sp, tile_ns.get(nm, max(500, est)),
                                 gemm_tile_bytes(n, k // sp), measured_time=measured.get(nm)))
    ob = 26 if optim_mode == 0 else 18
    est = int(ob * 4096 * 3 / (6.5e12 / 147) * 1e9)
    specs.append(kernel_spec(optim_name, (pad_to(n_params, 4) + 4095) // 4096, tile_ns.get(optim_name, est),
                             ob * 4096 * 3, measured_time=measured.get(optim_name)))
    return specs, sequence


class TrainStepLP:
    """One LP tenant = one training step: every distinct GEMM shape of the step registered
    once as a preemptible tcgen05 LP kernel (shared scratch operands), plus the optimizer
    streamer.  `sequence` is the step's kernel order as (name, repeat) runs — the LP task's
    kernel_sequence in the scenario (model.hpp KernelRef) — so the live runtime issues the
    step's GEMMs in order, each one a parent whose tiles are harvested / preempted."""

    def __init__(self, dev: Device, prefix: str, gemms: list[tuple[str, int, int, int]], n_params: int,
                 optim_mode: int, seed: int, tensor_base: int):
        self.dev, self.prefix, self.gemms, self.optim_mode = dev, prefix, gemms, optim_mode
        by_name, self.sequence, self.optim_name = step_plan(prefix, gemms, optim_mode)
        shapes = {shp: nm for nm, shp in by_name.items()}
        amax = max(m * k for m, n, k in shapes)
        bmax = max(n * k for m, n, k in shapes)
        cmax = max(m * n for m, n, k in shapes)
        self.scratch = [dev.alloc(2 * x) for x in (amax, bmax, cmax)]
        dev.fill_synth(self.scratch[0], amax, seed, tensor_base + 1, 1.0)
        dev.fill_synth(self.scratch[1], bmax, seed, tensor_base + 2, 0.02)
        self.kernels: dict[str, object] = {}
        self.shape: dict[str, tuple[int, int, int]] = {}
        self.flops = 0
        for (m, n, k), nm in shapes.items():
            self.kernels[nm] = dev.lp_register_gemm(self.scratch[0], self.scratch[1], self.scratch[2], m, n, k,
                                                     block_n=block_n_for(n), split_k=split_for(m, n, k))
            self.shape[nm] = (m, n, k)
        for _, m, n, k in gemms:
            self.flops += 2 * m * n * k
        # optimizer: fp32 master params / moments, bf16 grads
        self.n_params = pad_to(n_params, 4)
        np_ = self.n_params
        self.opt_bufs = [dev.alloc(4 * np_), dev.alloc(4 * np_), dev.alloc(4 * np_) if optim_mode == 0 else 0,
                         dev.alloc(2 * np_)]
        dev.fill_synth_f32(self.opt_bufs[0], np_, seed, tensor_base + 3, 0.05)
        dev.memset(self.opt_bufs[1], 0, 4 * np_)
        if optim_mode == 0:
            dev.memset(self.opt_bufs[2], 0, 4 * np_)
        dev.fill_synth(self.opt_bufs[3], np_, seed, tensor_base + 4, 0.01)
        if optim_mode == 0:
            self.kernels[self.optim_name] = dev.lp_register_optim(*self.opt_bufs, np_, mode=0, lr=1e-4, beta1=0.9,
                                                                  beta2=0.999, eps=1e-8, wd=0.01, c1=10.0,
                                                                  c2=1000.0)
        else:
            self.kernels[self.optim_name] = dev.lp_register_optim(self.opt_bufs[0], self.opt_bufs[1], 0,
                                                                  self.opt_bufs[3], np_, mode=1, lr=0.1, beta1=0.9,
                                                                  wd=1e-4)
        self.tile_ns: dict[str, int] = {}
        self.measured: dict[str, list] = {}

    def binding(self) -> dict:
        return {nm: k.id for nm, k in self.kernels.items()}

    def calibrate(self, reps: int = 2) -> dict:
        """Per-kernel full-run time (CUDA events) -> per-wave tile time of the pacing model
        (the on-B200 profile behind KernelSpec.block_time)."""
        self.dev.set_lp_sm_reserve(1)  # a live run may have left a governed reserve
        sm = self.dev.info["sm_count"] - 1
        self.ms: dict[str, float] = {}
        for nm, k in self.kernels.items():
            ms = self.dev.lp_time_full(k, reps)
            self.ms[nm] = ms
            resident = (sm // k.tile_ctas) if nm != self.optim_name else 3 * sm
            waves = math.ceil(k.total_tiles / resident)
            self.tile_ns[nm] = max(500, int(ms * 1e6 / max(1, waves)))
            # two-point on-B200 profile (one wave, whole kernel) -> KernelSpec.measured_time
            rows = [(k.total_tiles, int(ms * 1e6))]
            if k.total_tiles > resident:
                rows.insert(0, (resident, int(self.dev.lp_time_range(k, 0, resident, 1) * 1e6)))
            self.measured[nm] = [{"n_blocks": int(n), "time": {"value": max(1, t), "unit": "ns"}} for n, t in rows]
        self.step_ms = sum(self.ms[nm] * r for nm, r in self.sequence)
        return {"step_ms": self.step_ms, "kernels": len(self.kernels), "gemm_tflop_per_step": self.flops / 1e12,
                "gemm_tflops": self.flops / (sum(self.ms[nm] * r for nm, r in self.sequence
                                                 if nm != self.optim_name) * 1e-3) / 1e12}

    def kernel_specs(self) -> list[dict]:
        """Reference-schema KernelSpecs of the step's kernels with the measured tile times
        (grids = this device's tile counts)."""
        specs, _ = step_specs(self.prefix, self.gemms, self.n_params, self.optim_mode, self.tile_ns, self.measured)
        for sp in specs:
            assert sp["grid"][0] == self.kernels[sp["name"]].total_tiles, sp["name"]
        return specs

    def free(self):
        for k in self.kernels.values():
            self.dev.lp_unregister(k)
        for p in self.scratch + [b for b in self.opt_bufs if b]:
            self.dev.free(p)
        self.kernels.clear()
