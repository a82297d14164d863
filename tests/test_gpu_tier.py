"""Live memory tier on B200 (include/ms_tier.h): LP buffers that
overflow the tier's HBM budget spill 2 MB chunks to host DRAM (no NVLink peer on a 1-GPU
box) inside ONE virtual range, the unmodified preemptible LP streamer computes on them
bit-exactly, and an HP allocation displaces LP chunks (priority isolation) without
changing a byte the LP tenant sees.  Placement decisions = MemoryManager (the replay
engine's code, parity-tested against the reference in test_replay_parity.py)."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
CHUNK = 2 << 20


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


def run_preempted(dev, k, preemptions=3):
    begin = 0
    for i in range(100):
        dev.lp_run(k, begin, k.total_tiles)
        if i < preemptions:
            time.sleep(50e-6)
            dev.preempt_raise()
        st = dev.lp_wait(k, 60)
        begin = min(st["cursor"], k.total_tiles)
        if begin >= k.total_tiles and st["redo_count"] == 0:   # parked units drained too
            return i + 1
    raise AssertionError("LP run did not finish")


def test_tier_spill_relocation_and_axpy_exact(dev):
    from oracle import tenant as T
    from paper_2601_04071_b200.tier import MemoryTier
    n = 1 << 26                                  # 128 MB per bf16 tensor = 64 chunks
    budget_chunks = int(0.2e9 // CHUNK)          # 95
    with MemoryTier(dev, {"hbm_gb": 0.2}) as tier:
        x = tier.alloc(1, 2 * n)
        y = tier.alloc(1, 2 * n)
        cx, cy = tier.chunks(x), tier.chunks(y)
        assert [c[0] for c in cx] == ["local"] * 64
        n_local_y = budget_chunks - 64
        assert [c[0] for c in cy] == ["local"] * n_local_y + ["dram"] * (64 - n_local_y)
        assert not any(c[3] for c in cx + cy)
        st = tier.stats()
        assert st["local_used_chunks"] == budget_chunks and st["chunks_dram"] == 64 - n_local_y

        dev.fill_synth(x, n, 9, 1, 1.0)
        dev.fill_synth(y, n, 9, 2, 1.0)
        xs, ys = T.synth_bf16(n, 9, 1, 1.0), T.synth_bf16(n, 9, 2, 1.0)
        k = dev.lp_register_axpy(x, y, n, 1.5)
        assert run_preempted(dev, k) > 1
        want = T.axpy(ys, xs, 1.5)
        assert np.array_equal(d2h(dev, y, n), want)

        # HP allocation with the budget full: pinned local, displaces the 40 oldest LP chunks
        h = tier.alloc(0, 40 * CHUNK, high_priority=True)
        assert all(c == ("local", -1, 0, True) for c in tier.chunks(h))
        cx = tier.chunks(x)
        assert [c[0] for c in cx[:40]] == ["dram"] * 40 and [c[0] for c in cx[40:]] == ["local"] * 24
        st = tier.stats()
        assert st["relocations"] == 40 and st["relocated_bytes"] == 40 * CHUNK
        assert np.array_equal(d2h(dev, x, n), xs)     # relocation preserved every byte
        assert np.array_equal(d2h(dev, y, n), want)

        dev.memset(h, 0x5A, 40 * CHUNK)               # HP writes its own chunks only
        dev.lp_reset(k)
        run_preempted(dev, k, preemptions=1)
        assert np.array_equal(d2h(dev, y, n), T.axpy(want, xs, 1.5))
        assert np.array_equal(d2h(dev, x, n), xs)
        # bounded off-device admission: same bytes, preempted mid-run
        slow = tier.off_device(x, y)
        assert sum(slow) == len(set(range(40)) | set(range(n_local_y, 64)))
        ys2 = d2h(dev, y, n)
        dev.lp_set_slow_tiles(k, slow, CHUNK // (2 * 8192), 2)
        dev.lp_reset(k)
        assert run_preempted(dev, k, preemptions=4) > 1
        assert np.array_equal(d2h(dev, y, n), T.axpy(ys2, xs, 1.5))
        with pytest.raises(Exception, match="cover"):
            dev.lp_set_slow_tiles(k, slow[:3], CHUNK // (2 * 8192), 2)
        dev.lp_set_slow_tiles(k, None, 0)
        dev.lp_unregister(k)
        for p in (x, y, h):
            tier.free(p)
        assert tier.stats()["local_used_chunks"] == 0


def test_tier_errors(dev):
    from paper_2601_04071_b200.device import DeviceError
    from paper_2601_04071_b200.tier import MemoryTier
    with pytest.raises(DeviceError, match="eviction"):
        MemoryTier(dev, {"eviction": "lru"})
    with pytest.raises(DeviceError, match="P2P peer"):
        MemoryTier(dev, {"peers": [{"device": 0, "free_gb": 1.0}]})
    with MemoryTier(dev, {"hbm_gb": 0.01}) as tier:   # 4 chunks
        with pytest.raises(DeviceError, match="no such link"):
            tier.probe(0)
        tier.alloc(0, 4 * CHUNK, high_priority=True)
        with pytest.raises(DeviceError, match="exhausted by pinned"):
            tier.alloc(0, CHUNK, high_priority=True)


@pytest.mark.parametrize("pair", [0, 1])
def test_tier_gemm_operand_admission(dev, pair):
    """GEMM operands partly in host DRAM (the tier spilled them): with the per-unit slow map
    (tier.gemm_slow_units) the LP GEMM — single-CTA (tc_gemm.cuh) or on CTA pairs
    (tc_gemm2.cuh) — admits at most 2 off-device units at once, and preempted + resumed runs
    stay bit-identical to an unconstrained run from HBM."""
    import os
    from paper_2601_04071_b200.tier import MemoryTier
    m, n, k = 4096, 2048, 8192                  # A 64 MB = 32 chunks, B 32 MB = 16 chunks
    with MemoryTier(dev, {"hbm_gb": 0.08}) as tier:   # 38 chunks: B spills 10
        a = tier.alloc(1, m * k * 2)
        b = tier.alloc(1, n * k * 2)
        c = dev.alloc(m * n * 2)
        dev.fill_synth(a, m * k, 11, 1, 1.0)
        dev.fill_synth(b, n * k, 11, 2, 1.0 / 90.5)
        assert any(x[0] == "dram" for x in tier.chunks(b))
        os.environ["MS_LP_GEMM_PAIR"] = str(2 * pair)
        try:
            kern = dev.lp_register_gemm(a, b, c, m, n, k, block_n=256)
        finally:
            os.environ.pop("MS_LP_GEMM_PAIR")
        assert kern.tile_ctas == 1 + pair
        dev.lp_run(kern, 0, kern.total_tiles)
        dev.lp_wait(kern, 60)
        ref = d2h(dev, c, m * n)
        if pair:
            tn = n * (m // 256) // kern.total_tiles
            slow = tier.gemm_slow_units(a, b, m, n, k, block_m=256, block_n=tn, group_m=8)
        else:
            slow = tier.gemm_slow_units(a, b, m, n, k, block_n=256)
        assert len(slow) == kern.total_tiles and 0 < sum(slow) < len(slow)
        dev.lp_set_slow_tiles(kern, slow, 1, 2)
        dev.memset(c, 0, m * n * 2)
        dev.lp_reset(kern)
        assert run_preempted(dev, kern, preemptions=4) > 1
        assert np.array_equal(d2h(dev, c, m * n), ref)
        dev.lp_set_slow_tiles(kern, None, 0)
        dev.lp_unregister(kern)
        dev.free(c)
        for p in (a, b):
            tier.free(p)
