"""Property-based differential tests of every planning primitive against the compiled
reference (hypothesis drives the inputs)."""
from hypothesis import assume, given, settings, strategies as st

GPU = {"n_sm": 148, "sm_max_threads": 2048, "hbm_bandwidth": 6.5157e12,
       "launch_overhead": {"value": 7, "unit": "us"}, "sync_overhead": {"value": 5, "unit": "us"}}

u64 = st.integers(min_value=0, max_value=2**64 - 1)


@settings(max_examples=300, deadline=None)
@given(u64, u64)
def test_keyed_rng(ms, ref, a, b):
    assert ms.splitmix64(a) == ref.splitmix64(a)
    assert ms.hash_combine(a, b) == ref.hash_combine(a, b)
    assert ms.u01_from_key(a) == ref.u01_from_key(a)


@settings(max_examples=200, deadline=None)
@given(st.text(max_size=40))
def test_hash_str(ms, ref, s):
    assert ms.hash_str(s) == ref.hash_str(s)


kernels = st.builds(
    lambda gx, gy, tpb, occ, bt, bw, split: {
        "name": "k", "grid": [gx, gy, 1], "threads_per_block": tpb, "occupancy": occ,
        "block_time": {"dist": "point", "value": {"value": bt, "unit": "ns"}}, "bw_demand_per_block": bw,
        "splittable": split},
    st.integers(1, 300), st.integers(1, 40), st.sampled_from([64, 128, 256, 512]),
    st.sampled_from([1.0, 0.5, 0.25, 0.125]), st.integers(100, 2_000_000),
    st.sampled_from([0.0, 1e9, 2e10, 1e11]), st.just(True))


@settings(max_examples=150, deadline=None)
@given(kernels, st.integers(1, 20000), st.floats(0, 1e13), st.integers(0, 1))
def test_capacity_and_wave_model(ms, ref, k, n, load, rounding):
    assume(k["occupancy"] * 2048 >= k["threads_per_block"])  # KernelSpec::validate precondition
    assert ms.concurrent_capacity(GPU, k, rounding) == ref.concurrent_capacity(GPU, k, rounding)
    assert ms.exec_time_model(GPU, k, n, load, rounding) == ref.exec_time_model(GPU, k, n, load, rounding)


@settings(max_examples=150, deadline=None)
@given(kernels, st.sampled_from([0.0, 0.02, 0.1]), st.integers(1_000, 1_000_000), st.booleans())
def test_split_search(ms, ref, k, eps, cap, sq):
    assume(k["occupancy"] * 2048 >= k["threads_per_block"])
    a = ms.find_optimal_split(GPU, k, eps, cap, sq)
    b = ref.find_optimal_split(GPU, k, eps, cap, sq)
    assert a == b


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 50), st.integers(1, 20), st.integers(1, 5), st.integers(1, 6000), st.booleans())
def test_slices_and_consolidate(ms, ref, gx, gy, gz, bps, sq):
    a = ms.slice_boxes([gx, gy, gz], bps, sq)
    assert a == ref.slice_boxes([gx, gy, gz], bps, sq)
    # a random subset of the slices merges identically
    sub = a[::2]
    assert ms.consolidate([gx, gy, gz], sub) == ref.consolidate([gx, gy, gz], sub)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(1, 10**9), max_size=20), st.sampled_from([0.1, 0.3, 1.0]), st.integers(1, 10))
def test_predictor(ms, ref, gaps, alpha, k):
    assert ms.predict_interval(gaps, alpha, k) == ref.predict_interval(gaps, alpha, k)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(-10**12, 10**12), max_size=300), st.floats(0, 1))
def test_percentile(ms, ref, xs, q):
    assert ms.percentile(xs, q) == ref.percentile(xs, q)


@settings(max_examples=60, deadline=None)
@given(st.floats(0.5, 5000), st.floats(1.0, 8.0), st.integers(1, 2 * 10**9), u64)
def test_bursty_arrivals(ms, ref, rate, b, horizon, seed):
    assert ms.generate_bursty_arrivals(rate, b, horizon, seed) == ref.generate_bursty_arrivals(rate, b, horizon, seed)


@settings(max_examples=80, deadline=None)
@given(kernels, st.lists(st.integers(1, 4000), min_size=1, max_size=30), st.integers(1, 10**8),
       st.sampled_from([1.0, 1.2, 3.0]))
def test_consolidation_prefix(ms, ref, k, blocks, interval, safety):
    assume(k["occupancy"] * 2048 >= k["threads_per_block"])
    assert ms.consolidation_prefix(GPU, k, blocks, interval, safety) == \
        ref.consolidation_prefix(GPU, k, blocks, interval, safety)
