"""Preemption semantics on B200: preempt mid-run, record the cursor, resume from it —
the final result must equal the uninterrupted run bit-exactly (GEMM and streamer), the
harvest budget must bound the run, and flag -> exit latency must stay µs-scale."""
import math
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2601_04071_b200.device import Device
    d = Device(0)
    yield d
    d.close()


def d2h(dev, ptr, n):
    out = np.empty(n, np.uint16)
    dev.d2h(out.ctypes.data, ptr, n * 2)
    return out


def spin(seconds):
    t = time.perf_counter() + seconds
    while time.perf_counter() < t:
        pass


@pytest.fixture(scope="module")
def gemm(dev):
    n = 4096
    a, b, c = dev.alloc(n * n * 2), dev.alloc(n * n * 2), dev.alloc(n * n * 2)
    dev.fill_synth(a, n * n, 5, 1, 1.0)
    dev.fill_synth(b, n * n, 5, 2, float(np.float32(1 / math.sqrt(n))))
    k = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
    dev.lp_run(k, 0, k.total_tiles)
    dev.lp_wait(k, 30)
    return n, c, k, d2h(dev, c, n * n)


def test_gemm_preempt_resume_bit_exact(dev, gemm):
    n, c, k, ref = gemm
    off, _ = dev.calibrate(100)
    # A preemption lands ~5 us after the raise; runs shorter than one tile (~30 us here)
    # complete nothing (abandoned tiles restart), so every run gets at least ~1 tile time.
    for delay in (40e-6, 70e-6):  # the whole 4096^3 GEMM takes ~105 us
        dev.memset(c, 0, n * n * 2)
        dev.lp_reset(k)
        begin, runs, exits = 0, 0, []
        while True:
            dev.lp_run(k, begin, k.total_tiles)
            runs += 1
            spin(delay)
            _, t_raise = dev.preempt_raise()
            st = dev.lp_wait(k, 30)
            if st["preempted"]:
                exits.append(st["t_exit"] - off - t_raise)
            assert st["cursor"] >= begin
            begin = st["cursor"]
            if begin >= k.total_tiles and st["redo_count"] == 0:
                break
            assert runs < 3000
        assert runs > 1
        assert np.array_equal(d2h(dev, c, n * n), ref), delay
        if exits:
            assert sorted(exits)[len(exits) // 2] < 100_000   # µs-scale drain (loose CI bound)


def test_budget_bounds_the_run(dev, gemm):
    n, c, k, ref = gemm
    dev.lp_reset(k)
    budget = k.total_tiles // 2
    dev.lp_run(k, 0, k.total_tiles, budget=budget)
    st = dev.lp_wait(k, 30)
    assert not st["preempted"]
    done_fresh = st["tiles_done"]
    assert st["cursor"] >= budget and done_fresh <= budget + 148
    # the rest of the range, including parked tiles, completes the GEMM exactly
    dev.lp_run(k, st["cursor"], k.total_tiles)
    st2 = dev.lp_wait(k, 30)
    assert st2["cursor"] == k.total_tiles and st2["redo_count"] == 0
    assert st["tiles_done"] + st2["tiles_done"] == k.total_tiles
    assert np.array_equal(d2h(dev, c, n * n), ref)


@pytest.mark.parametrize("pair", [0, 1, 2])  # single CTA / pairs with 256 x 256 / 256 x 512 tiles
def test_gemm_cta_pair_kernel_preempt_resume(dev, pair):
    """The cta_group::2 LP GEMM (MS_LP_GEMM_PAIR=1, tc_gemm2.cuh) and the single-CTA one
    produce the same bits, uninterrupted and preempted + resumed."""
    import os
    n = 2048
    a, b, c = dev.alloc(n * n * 2), dev.alloc(n * n * 2), dev.alloc(n * n * 2)
    dev.fill_synth(a, n * n, 8, 1, 1.0)
    dev.fill_synth(b, n * n, 8, 2, float(np.float32(1 / math.sqrt(n))))
    old = os.environ.get("MS_LP_GEMM_PAIR")
    os.environ["MS_LP_GEMM_PAIR"] = str(pair)
    try:
        k = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
    finally:
        if old is None:
            os.environ.pop("MS_LP_GEMM_PAIR")
        else:
            os.environ["MS_LP_GEMM_PAIR"] = old
    assert k.total_tiles == {0: (n // 128) * (n // 256), 1: (n // 256) ** 2, 2: (n // 256) * (n // 512)}[pair]
    dev.lp_run(k, 0, k.total_tiles)
    dev.lp_wait(k, 30)
    ref = d2h(dev, c, n * n)
    dev.memset(c, 0, n * n * 2)
    dev.lp_reset(k)
    begin, runs = 0, 0
    while True:
        dev.lp_run(k, begin, k.total_tiles)
        runs += 1
        # raised at different points of the run: the pair's two producers then stop at
        # different k-blocks in either order (tc_gemm2.cuh stop agreement)
        spin((2e-6, 15e-6, 40e-6, 7e-6)[runs % 4])
        dev.preempt_raise()
        st = dev.lp_wait(k, 30)
        begin = st["cursor"]
        if begin >= k.total_tiles and st["redo_count"] == 0:
            break
        assert runs < 3000
    assert np.array_equal(d2h(dev, c, n * n), ref)
    if pair:  # same bits as the single-CTA kernel
        os.environ.pop("MS_LP_GEMM_PAIR", None)
        k1 = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
        dev.memset(c, 0, n * n * 2)
        dev.lp_run(k1, 0, k1.total_tiles)
        dev.lp_wait(k1, 30)
        assert np.array_equal(d2h(dev, c, n * n), ref)
        dev.lp_unregister(k1)
    dev.lp_unregister(k)
    for p_ in (a, b, c):
        dev.free(p_)


@pytest.mark.parametrize("ctas_per_sm", [4, 1])  # 1 = grouped one-CTA-per-SM streamer
def test_axpy_preempt_resume_exact(dev, ctas_per_sm):
    from oracle import tenant as T
    n = 1 << 26
    x, y = dev.alloc(2 * n), dev.alloc(2 * n)
    dev.fill_synth(x, n, 3, 1, 1.0)
    dev.fill_synth(y, n, 3, 2, 1.0)
    k = dev.lp_register_axpy(x, y, n, 1.5, ctas_per_sm=ctas_per_sm)
    begin, runs = 0, 0
    while True:
        dev.lp_run(k, begin, k.total_tiles)
        runs += 1
        spin(20e-6)
        dev.preempt_raise()
        st = dev.lp_wait(k, 30)
        assert st["redo_count"] == 0          # streamer tiles are never abandoned mid-tile
        begin = st["cursor"]
        if begin >= k.total_tiles:
            break
    assert runs > 1
    want = T.axpy(T.synth_bf16(n, 3, 2, 1.0), T.synth_bf16(n, 3, 1, 1.0), 1.5)
    assert np.array_equal(d2h(dev, y, n), want)
    dev.lp_unregister(k)
    dev.free(x)
    dev.free(y)


def test_doorbell_releases_armed_chain(dev):
    M, H = 128, 1024
    a, w, c = dev.alloc(M * H * 2), dev.alloc(H * H * 2), dev.alloc(M * H * 2)
    dev.fill_synth(a, M * H, 1, 1, 1.0)
    dev.fill_synth(w, H * H, 1, 2, 1 / 32)
    chain = dev.hp_register_chain([dict(kind=1, block_n=64, a=a, b=w, c=c, bias=0, m=M, n=H, k=H)])
    seq = dev.hp_next_seq()
    dev.hp_arm(chain, seq)
    time.sleep(0.02)
    assert dev.hp_poll(chain, seq) is None        # held at the gate until the ring
    dev.hp_ring(seq)
    t = dev.hp_wait(chain, seq, 10)
    assert t["done"] and t["t_done"] >= t["t_first_cta"] >= t["t_gate"] > 0
