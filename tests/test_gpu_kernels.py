"""Tenant-kernel numeric parity on B200 (north_star: fp32 rel <= 1e-3, bf16 rel <= 1e-2)
against the C restatement in oracle/tenant_ref.c, all through the C-ABI."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
BF16_TOL = 1e-2  # bf16 outputs (north_star)
SEED = 99


@pytest.fixture(scope="module")
def dev():
    from paper_2601_04071_b200.device import Device
    d = Device(0)
    yield d
    d.close()


@pytest.fixture(scope="module")
def T():
    from oracle import tenant
    return tenant


def d2h(dev, ptr, n):
    out = np.empty(n, np.uint16)
    dev.d2h(out.ctypes.data, ptr, n * 2)
    return out


def test_synthetic_generator_is_bit_identical(dev, T):
    n = 1 << 20
    p = dev.alloc(2 * n)
    for tensor, scale in ((1, 1.0), (9, 0.03125), (77, float(np.float32(1 / math.sqrt(4096))))):
        dev.fill_synth(p, n, SEED, tensor, scale)
        assert np.array_equal(d2h(dev, p, n), T.synth_bf16(n, SEED, tensor, scale))
    dev.free(p)


@pytest.mark.parametrize("M,N,K,bn", [(128, 256, 64, 256), (256, 512, 320, 256), (384, 384, 1024, 128),
                                      (128, 1024, 512, 64), (1024, 2048, 2048, 256)])
def test_gemm_matches_oracle(dev, T, M, N, K, bn):
    a, b, c = dev.alloc(M * K * 2), dev.alloc(N * K * 2), dev.alloc(M * N * 2)
    s = float(np.float32(1 / math.sqrt(K)))
    dev.fill_synth(a, M * K, SEED, 1, 1.0)
    dev.fill_synth(b, N * K, SEED, 2, s)
    dev.memset(c, 0xFF, M * N * 2)
    k = dev.lp_register_gemm(a, b, c, M, N, K, block_n=bn)
    dev.lp_run(k, 0, k.total_tiles)
    st = dev.lp_wait(k, 30)
    assert st["tiles_done"] == k.total_tiles and st["cursor"] == k.total_tiles and st["redo_count"] == 0
    rows = list(range(M)) if M <= 384 else list(range(0, M, 7))
    want = T.gemm_rows(T.synth_bf16(M * K, SEED, 1, 1.0), T.synth_bf16(N * K, SEED, 2, s), rows, N, K)
    got = T.bf16_to_f32(d2h(dev, c, M * N).reshape(M, N)[rows].reshape(-1)).reshape(len(rows), N)
    rel = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert rel <= BF16_TOL, rel
    dev.lp_unregister(k)
    for p in (a, b, c):
        dev.free(p)


def test_gemm_8192_sampled_tiles(dev, T):
    """Full config-1 LP GEMM; >= 64 sampled output rows spanning every M tile."""
    n = 8192
    a, b, c = dev.alloc(n * n * 2), dev.alloc(n * n * 2), dev.alloc(n * n * 2)
    s = float(np.float32(1 / math.sqrt(n)))
    dev.fill_synth(a, n * n, SEED, 1, 1.0)
    dev.fill_synth(b, n * n, SEED, 2, s)
    k = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
    dev.lp_run(k, 0, k.total_tiles)
    dev.lp_wait(k, 60)
    rows = [t * 128 + (t * 37) % 128 for t in range(64)]
    want = T.gemm_rows(T.synth_bf16(n * n, SEED, 1, 1.0), T.synth_bf16(n * n, SEED, 2, s), rows, n, n)
    C = d2h(dev, c, n * n).reshape(n, n)
    got = T.bf16_to_f32(C[rows].reshape(-1)).reshape(len(rows), n)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= BF16_TOL
    dev.lp_unregister(k)
    for p in (a, b, c):
        dev.free(p)


@pytest.mark.parametrize("n,tile", [(1 << 20, 8192), (3 * 8192 + 8 * 5, 2048), (1 << 24, 16384)])
def test_axpy_bit_exact(dev, T, n, tile):
    x, y = dev.alloc(2 * n), dev.alloc(2 * n)
    dev.fill_synth(x, n, SEED, 11, 1.0)
    dev.fill_synth(y, n, SEED, 12, 1.0)
    k = dev.lp_register_axpy(x, y, n, -0.375, tile_elems=tile)
    dev.lp_run(k, 0, k.total_tiles)
    dev.lp_wait(k, 30)
    want = T.axpy(T.synth_bf16(n, SEED, 12, 1.0), T.synth_bf16(n, SEED, 11, 1.0), -0.375)
    assert np.array_equal(d2h(dev, y, n), want)
    dev.lp_unregister(k)
    dev.free(x)
    dev.free(y)


@pytest.mark.parametrize("fused", [1, 2, 0])
def test_hp_chain_matches_oracle(dev, T, fused):
    """Config-1 HP chain: 4 chained GEMMs + bias/GELU; fp32-accumulated bf16 ops — as one
    fused launch (cluster/DSMEM split-K, or global split-K) and as one kernel per op."""
    dev.hp_set_fused(fused)
    M, H = 128, 1024
    act = [dev.alloc(M * H * 2) for _ in range(5)]
    ws = [dev.alloc(H * H * 2) for _ in range(4)]
    bias = dev.alloc(H * 2)
    s = float(np.float32(1 / math.sqrt(H)))
    dev.fill_synth(act[0], M * H, SEED, 100, 1.0)
    for i, w in enumerate(ws):
        dev.fill_synth(w, H * H, SEED, 101 + i, s)
    dev.fill_synth(bias, H, SEED, 110, 0.1)
    ops = [dict(kind=1, block_n=64, a=act[i], b=ws[i], c=act[i + 1], bias=0, m=M, n=H, k=H) for i in range(4)]
    out = dev.alloc(M * H * 2)
    ops.append(dict(kind=2, block_n=0, a=act[4], b=0, c=out, bias=bias, m=M, n=H, k=0))
    chain = dev.hp_register_chain(ops)
    dev.hp_launch_direct(chain, dev.hp_next_seq())
    dev.sync()
    x = T.synth_bf16(M * H, SEED, 100, 1.0)
    for i in range(4):   # oracle chain, rounding to bf16 between ops like the device does
        y = T.gemm_rows(x, T.synth_bf16(H * H, SEED, 101 + i, s), list(range(M)), H, H).reshape(-1)
        x = np.ascontiguousarray((y.view(np.uint32) + 0x7FFF + ((y.view(np.uint32) >> 16) & 1)) >> 16).astype(np.uint16)
        got_i = T.bf16_to_f32(d2h(dev, act[i + 1], M * H))
        ref_i = T.bf16_to_f32(x)
        assert np.max(np.abs(got_i - ref_i)) / np.max(np.abs(ref_i)) <= BF16_TOL, i
    want = T.bf16_to_f32(T.bias_gelu(d2h(dev, act[4], M * H), T.synth_bf16(H, SEED, 110, 0.1), M, H))
    got = T.bf16_to_f32(d2h(dev, out, M * H))
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= BF16_TOL
    dev.hp_set_fused(True)


def test_hp_silu_mul_matches_oracle(dev, T):
    """Standalone SILU_MUL op (fused and per-op): out = silu(gate) * up over [M x 2N]."""
    M, N = 256, 1024
    x, out = dev.alloc(M * 2 * N * 2), dev.alloc(M * N * 2)
    dev.fill_synth(x, M * 2 * N, SEED, 41, 2.0)
    want = T.bf16_to_f32(T.silu_mul(T.synth_bf16(M * 2 * N, SEED, 41, 2.0), M, N))
    for fused in (1, 0):
        dev.hp_set_fused(fused)
        dev.memset(out, 0, M * N * 2)
        ch = dev.hp_register_chain([dict(kind=5, block_n=0, a=x, b=0, c=out, bias=0, m=M, n=N, k=0)])
        dev.hp_launch_direct(ch, dev.hp_next_seq())
        dev.sync()
        got = T.bf16_to_f32(d2h(dev, out, M * N))
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= BF16_TOL
        dev.hp_unregister_chain(ch)
    dev.hp_set_fused(1)


def test_hp_chain_fused_equals_per_op(dev, T):
    """Per-op kernels, the cluster (DSMEM) fused launch and the global-reduction fused
    launch use the same tiles, k-slices and slice-order sums: config-1-size chains agree
    bit for bit (and across repeated launches).  The opt-in narrow plan (128 x 32 tiles, whole
    K in one accumulator) rounds differently: bf16 tolerance, and bit-identical across its own
    repeated launches."""
    import os
    M, H = 128, 4096
    act = [dev.alloc(M * H * 2) for _ in range(5)]
    ws = [dev.alloc(H * H * 2) for _ in range(4)]
    bias, out = dev.alloc(H * 2), dev.alloc(M * H * 2)
    s = float(np.float32(1 / math.sqrt(H)))
    for i, w in enumerate(ws):
        dev.fill_synth(w, H * H, SEED, 201 + i, s)
    dev.fill_synth(bias, H, SEED, 210, 0.1)
    ops = [dict(kind=1, block_n=128, a=act[i], b=ws[i], c=act[i + 1], bias=0, m=M, n=H, k=H) for i in range(4)]
    ops.append(dict(kind=2, block_n=0, a=act[4], b=0, c=out, bias=bias, m=M, n=H, k=0))
    def run(fused, narrow):
        os.environ["MS_FUSED_NARROW"] = "1" if narrow else "0"
        try:
            dev.hp_set_fused(fused)
            chain = dev.hp_register_chain(ops)
        finally:
            os.environ.pop("MS_FUSED_NARROW", None)
        info = dev.hp_chain_info(chain)
        assert info["fused_grid"] == 128
        if fused:
            assert info["cluster"] == (4 if (fused == 1 and not narrow) else 1)
        dev.fill_synth(act[0], M * H, SEED, 200, 1.0)
        for a in act[1:] + [out]:
            dev.memset(a, 0, M * H * 2)
        dev.hp_launch_direct(chain, dev.hp_next_seq())
        dev.sync()
        dev.hp_unregister_chain(chain)
        return [d2h(dev, a, M * H) for a in act[1:] + [out]]

    results = [run(0, False), run(1, False), run(1, False), run(2, False)]
    narrow = [run(1, True), run(1, True)]
    dev.hp_set_fused(True)
    for r in results[1:]:
        for x, y in zip(results[0], r):
            assert np.array_equal(x, y)
    for x, y in zip(narrow[0], narrow[1]):
        assert np.array_equal(x, y)
    for x, y in zip(results[0], narrow[0]):
        fx, fy = T.bf16_to_f32(x), T.bf16_to_f32(y)
        assert np.max(np.abs(fx - fy)) / np.max(np.abs(fx)) <= BF16_TOL


@pytest.mark.parametrize("split", [1, 2, 4, 8])
def test_hp_gemm_split_k_matches_oracle(dev, T, split):
    """Skinny HP GEMM (M=128) with k-slices reduced in slice order by the last unit."""
    M, N, K = 128, 2048, 4096
    a, w, c = dev.alloc(M * K * 2), dev.alloc(N * K * 2), dev.alloc(M * N * 2)
    s = float(np.float32(1 / math.sqrt(K)))
    dev.fill_synth(a, M * K, SEED, 31, 1.0)
    dev.fill_synth(w, N * K, SEED, 32, s)
    chain = dev.hp_register_chain([dict(kind=1, block_n=128, a=a, b=w, c=c, bias=0, m=M, n=N, k=K, split_k=split)])
    for _ in range(2):  # second launch reuses the self-resetting tile counters
        dev.memset(c, 0, M * N * 2)
        dev.hp_launch_direct(chain, dev.hp_next_seq())
        dev.sync()
    want = T.gemm_rows(T.synth_bf16(M * K, SEED, 31, 1.0), T.synth_bf16(N * K, SEED, 32, s), list(range(M)), N, K)
    got = T.bf16_to_f32(d2h(dev, c, M * N)).reshape(M, N)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= BF16_TOL


DECODE_SMALL = (256, 384, 512, 1024, 2)          # H, Q, F, V, layers
DECODE_LLAMA = (2048, 3072, 8192, 4096, 1)       # Llama-3.2-1B layer geometry, short vocab


@pytest.mark.parametrize("M,fused,geom", [(128, 1, DECODE_SMALL), (128, 2, DECODE_SMALL), (128, 0, DECODE_SMALL),
                                          (1, 1, DECODE_SMALL), (1, 1, DECODE_LLAMA)])
def test_hp_decode_chain_matches_oracle(dev, T, M, fused, geom):
    """Config-4 HP step (layers + LM head) incl. strided A and the fused GEMM+SwiGLU op,
    against the oracle chain with bf16 rounding between ops.  M = 128: tcgen05 chain;
    M = 1 (bs=1 decode): the HBM-streaming GEMV chain (hp_gemv.cuh)."""
    dev.hp_set_fused(fused)
    H, Q, F, V, L = geom
    bufs = [dev.alloc(M * n * 2) for n in (H, Q, H, 2 * F, F, V)]
    s = lambda k: float(np.float32(1 / math.sqrt(k)))
    ws, host_w = [], []
    for l in range(L):
        shapes = [(Q, H), (H, H), (2 * F, H), (H, F)]
        ptrs = []
        hw = []
        for j, (n, k) in enumerate(shapes):
            p = dev.alloc(n * k * 2)
            dev.fill_synth(p, n * k, SEED, 300 + 10 * l + j, s(k))
            ptrs.append(p)
            hw.append(T.synth_bf16(n * k, SEED, 300 + 10 * l + j, s(k)))
        ws.append(ptrs)
        host_w.append(hw)
    lm = dev.alloc(V * H * 2)
    dev.fill_synth(lm, V * H, SEED, 399, s(H))
    dev.fill_synth(bufs[0], M * H, SEED, 298, 1.0)
    from paper_2601_04071_b200.live import decode_step_ops
    chain = dev.hp_register_chain(decode_step_ops(M, H, Q, F, V, L, bufs, ws, lm))
    if M == 1:
        ci = dev.hp_chain_info(chain)
        assert ci["fused_grid"] == dev.info["sm_count"] - 1 and ci["cluster"] == 1
    for _ in range(2):  # a second launch must reproduce the first (phase counters reset)
        dev.sync()
        dev.fill_synth(bufs[0], M * H, SEED, 298, 1.0)  # the chain overwrites h
        dev.hp_launch_direct(chain, dev.hp_next_seq())
    dev.sync()

    def rnd(y):  # fp32 -> bf16 bits (RNE), like the device epilogue
        u = y.astype(np.float32).view(np.uint32)
        return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)

    rows = list(range(M))
    h = T.synth_bf16(M * H, SEED, 298, 1.0)
    for l in range(L):
        wq, wo, wg, wd = host_w[l]
        qkv = rnd(T.gemm_rows(h, wq, rows, Q, H).reshape(-1))
        qh = np.ascontiguousarray(qkv.reshape(M, Q)[:, :H]).reshape(-1)
        o = rnd(T.gemm_rows(qh, wo, rows, H, H).reshape(-1))
        gu = T.gemm_rows(o, wg, rows, 2 * F, H)  # fp32 gate|up: the SwiGLU acts on the accumulators
        g, u = gu[:, :F], gu[:, F:]
        act = rnd((g / (1.0 + np.exp(-g)) * u).reshape(-1))
        h = rnd(T.gemm_rows(act, wd, rows, H, F).reshape(-1))
    want = T.gemm_rows(h, T.synth_bf16(V * H, SEED, 399, s(H)), rows, V, H)
    got = T.bf16_to_f32(d2h(dev, bufs[5], M * V)).reshape(M, V)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= BF16_TOL
    dev.hp_unregister_chain(chain)
    dev.hp_set_fused(1)


def test_hp_gemv_chain_elementwise_and_errors(dev, T):
    """Batch-1 chain with elementwise ops (GEMV -> BIAS_GELU -> GEMV -> SILU_MUL input), and
    the registration errors of the batch-1 path."""
    K, N = 512, 1000  # N not a multiple of the unit size: ragged last unit
    x, y0, y1, y2 = dev.alloc(K * 2), dev.alloc(N * 2), dev.alloc(N * 2), dev.alloc(2 * N * 2)
    w0, w1, bias = dev.alloc(N * K * 2), dev.alloc(2 * N * N * 2), dev.alloc(N * 2)
    s = lambda k: float(np.float32(1 / math.sqrt(k)))
    dev.fill_synth(x, K, SEED, 500, 1.0)
    dev.fill_synth(w0, N * K, SEED, 501, s(K))
    dev.fill_synth(w1, 2 * N * N, SEED, 502, s(N))
    dev.fill_synth(bias, N, SEED, 503, 0.1)
    ops = [dict(kind=1, block_n=0, a=x, b=w0, c=y0, bias=0, m=1, n=N, k=K),
           dict(kind=2, block_n=0, a=y0, b=0, c=y1, bias=bias, m=1, n=N, k=0),
           dict(kind=1, block_n=0, a=y1, b=w1, c=y2, bias=0, m=1, n=2 * N, k=N)]
    chain = dev.hp_register_chain(ops)
    dev.hp_launch_direct(chain, dev.hp_next_seq())
    dev.sync()
    h0 = T.gemm_rows(T.synth_bf16(K, SEED, 500, 1.0), T.synth_bf16(N * K, SEED, 501, s(K)), [0], N, K)
    u = h0.astype(np.float32).view(np.uint32)
    h0b = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16).reshape(-1)
    h1 = T.bias_gelu(h0b, T.synth_bf16(N, SEED, 503, 0.1), 1, N)
    got1 = d2h(dev, y1, N)
    assert np.max(np.abs(T.bf16_to_f32(got1) - T.bf16_to_f32(h1))) <= 2 * 2.0 ** -8 * np.max(np.abs(T.bf16_to_f32(h1)))
    want = T.gemm_rows(got1, T.synth_bf16(2 * N * N, SEED, 502, s(N)), [0], 2 * N, N)
    got = T.bf16_to_f32(d2h(dev, y2, 2 * N)).reshape(1, -1)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= BF16_TOL
    dev.hp_unregister_chain(chain)
    from paper_2601_04071_b200.device import DeviceError
    with pytest.raises(DeviceError):  # rows longer than one 16 KB stage
        dev.hp_register_chain([dict(kind=1, block_n=0, a=x, b=w0, c=y0, bias=0, m=1, n=8, k=16384)])
    with pytest.raises(DeviceError):  # m == 1 and m == 128 GEMMs in one chain
        dev.hp_register_chain([dict(kind=1, block_n=0, a=x, b=w0, c=y0, bias=0, m=1, n=128, k=512),
                               dict(kind=1, block_n=128, a=x, b=w0, c=y0, bias=0, m=128, n=128, k=512)])
    for p in (x, y0, y1, y2, w0, w1, bias):
        dev.free(p)
