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


@pytest.mark.parametrize("max_parts", [4, 2])
def test_gemm_pair_half_tail_units(dev, max_parts):
    """CTA pairs with 256 x 512 tiles: when the last wave is at most a quarter (half) full, its
    tiles run as four 128-column quarters (two 256-column halves) (tc_gemm2.cuh pair_unit;
    4864 x 2048 = 76 tiles on 73 pairs -> 73 full tiles + 12 quarter units, or 6 half units
    with MS_LP_PAIR_TAIL_PARTS=2).  Same bits as the single-CTA kernel, uninterrupted and
    preempted + resumed (part units parked on the redo list like tiles)."""
    import os
    from paper_2601_04071_b200.live import DEFAULT_LP_SM_RESERVE
    m, n, kk = 4864, 2048, 1024
    a, b, c = dev.alloc(m * kk * 2), dev.alloc(n * kk * 2), dev.alloc(m * n * 2)
    dev.fill_synth(a, m * kk, 9, 1, 1.0)
    dev.fill_synth(b, n * kk, 9, 2, float(np.float32(1 / math.sqrt(kk))))
    dev.set_lp_sm_reserve(DEFAULT_LP_SM_RESERVE)
    pairs = (dev.info["sm_count"] - ((DEFAULT_LP_SM_RESERVE + 1) & ~1)) // 2
    tiles = (m // 256) * (n // 512)
    tail = tiles % pairs
    os.environ["MS_LP_GEMM_PAIR"] = "2"
    os.environ["MS_LP_PAIR_TAIL_PARTS"] = str(max_parts)
    try:
        k = dev.lp_register_gemm(a, b, c, m, n, kk, block_n=256)
    finally:
        os.environ.pop("MS_LP_GEMM_PAIR")
        os.environ.pop("MS_LP_PAIR_TAIL_PARTS")
    assert k.tile_ctas == 2
    parts = 4 if max_parts == 4 and 4 * tail <= pairs else 2
    assert k.total_tiles == (tiles - tail + parts * tail if tiles >= pairs and 0 < 2 * tail <= pairs else tiles)
    assert k.total_tiles > tiles
    k1 = dev.lp_register_gemm(a, b, c, m, n, kk, block_n=256)  # single-CTA reference (pairs auto: too few tiles)
    assert k1.tile_ctas == 1
    dev.lp_run(k1, 0, k1.total_tiles)
    dev.lp_wait(k1, 30)
    ref = d2h(dev, c, m * n)
    dev.lp_unregister(k1)
    dev.memset(c, 0, m * n * 2)
    dev.lp_run(k, 0, k.total_tiles)
    st = dev.lp_wait(k, 30)
    assert st["tiles_done"] == k.total_tiles
    assert np.array_equal(d2h(dev, c, m * n), ref)
    dev.memset(c, 0, m * n * 2)
    dev.lp_reset(k)
    begin, runs = 0, 0
    while True:
        dev.lp_run(k, begin, k.total_tiles)
        runs += 1
        spin((3e-6, 20e-6, 60e-6, 9e-6)[runs % 4])
        dev.preempt_raise()
        st = dev.lp_wait(k, 30)
        begin = st["cursor"]
        if begin >= k.total_tiles and st["redo_count"] == 0:
            break
        assert runs < 3000
    assert np.array_equal(d2h(dev, c, m * n), ref)
    dev.lp_unregister(k)
    for p_ in (a, b, c):
        dev.free(p_)


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


def test_device_trace_ring(dev):
    """ms_trace_enable / ms_trace_drain: the kernels log their own exit records, HP chain
    completions and gate releases into a ring in pinned host memory, drained in order; a
    ring the host does not drain in time reports the overwritten events as lost."""
    import time as _t
    n = 2048
    a, b, c = dev.alloc(n * n * 2), dev.alloc(n * n * 2), dev.alloc(n * n * 2)
    dev.fill_synth(a, n * n, 8, 1, 1.0)
    dev.fill_synth(b, n * n, 8, 2, float(np.float32(1 / math.sqrt(n))))
    k = dev.lp_register_gemm(a, b, c, n, n, n, block_n=256)
    dev.trace_enable(1 << 12)
    dev.trace_drain()  # start from an empty window
    dev.lp_run(k, 0, k.total_tiles)
    spin(20e-6)
    dev.preempt_raise()
    st = dev.lp_wait(k, 30)
    dev.lp_run(k, st["cursor"], k.total_tiles)
    dev.lp_wait(k, 30)
    act = [dev.alloc(128 * 1024 * 2) for _ in range(2)]
    wgt = dev.alloc(1024 * 1024 * 2)
    dev.fill_synth(act[0], 128 * 1024, 7, 3, 1.0)
    dev.fill_synth(wgt, 1024 * 1024, 7, 4, 1 / 32)
    chain = dev.hp_register_chain([dict(kind=1, block_n=64, a=act[0], b=wgt, c=act[1], bias=0, m=128, n=1024, k=1024)])
    seq = dev.hp_next_seq()
    dev.hp_arm(chain, seq)
    _t.sleep(0.002)
    dev.hp_ring(seq)
    dev.hp_wait(chain, seq, 10)
    evs, lost = dev.trace_drain()
    assert lost == 0
    assert [e["seq"] for e in evs] == list(range(evs[0]["seq"], evs[0]["seq"] + len(evs)))
    lp = [e for e in evs if e["kind"] in ("lp_start", "lp_seen", "lp_exit") and e["id"] == k.id]
    exits = [e for e in lp if e["kind"] == "lp_exit"]
    assert len(exits) == 2 and len([e for e in lp if e["kind"] == "lp_start"]) == 2
    assert exits[0]["a"] < exits[1]["a"]  # run ids
    if st["preempted"]:
        seen = [e for e in lp if e["kind"] == "lp_seen"]
        assert len(seen) == 1 and seen[0]["a"] == exits[0]["a"] and seen[0]["t_ns"] <= exits[0]["t_ns"]
    assert (exits[0]["b"] >> 32) + (exits[1]["b"] >> 32) == k.total_tiles  # tiles done over both runs
    gate = [e for e in evs if e["kind"] == "gate" and e["id"] == seq]
    first = [e for e in evs if e["kind"] == "hp_first" and e["a"] == seq]
    done = [e for e in evs if e["kind"] == "hp_done" and e["a"] == seq]
    assert len(gate) == 1 and len(first) == 1 and len(done) == 1
    assert gate[0]["t_ns"] <= first[0]["t_ns"] <= done[0]["t_ns"]
    for _ in range(12):  # 12 unpreempted runs = 24 events, all held by the 4096-slot ring
        dev.lp_reset(k)
        dev.lp_run(k, 0, k.total_tiles)
        dev.lp_wait(k, 30)
    evs2, lost2 = dev.trace_drain()
    assert len(evs2) == 24 and lost2 == 0
    # overflow: a second device handle with a 16-slot ring, 24 events before the drain
    from paper_2601_04071_b200.device import Device
    d2 = Device(0)
    k2 = d2.lp_register_gemm(a, b, c, n, n, n, block_n=256)
    d2.trace_enable(16)
    for _ in range(12):
        d2.lp_reset(k2)
        d2.lp_run(k2, 0, k2.total_tiles)
        d2.lp_wait(k2, 30)
    evs3, lost3 = d2.trace_drain()
    assert len(evs3) == 16 and lost3 == 8 and evs3[0]["seq"] == 9 and evs3[-1]["seq"] == 24
    d2.lp_unregister(k2)
    d2.close()
    dev.trace_enable(0)
    dev.lp_reset(k)
    dev.lp_run(k, 0, k.total_tiles)
    dev.lp_wait(k, 30)
    assert dev.trace_drain()[0] == []  # disabled: nothing logged
    dev.hp_unregister_chain(chain)
    dev.lp_unregister(k)
    for p_ in (a, b, c, act[0], act[1], wgt):
        dev.free(p_)
