"""The sort path for two-word records (csrc/sort.cuh: one-sweep digit passes with
decoupled look-back, k_onesweep2; the fused segmented reduction, k_seg_emit2 /
k_seg_long2) against the numpy oracle: near-unique keys, long segments (a few
keys holding most records), segment lengths around the walk limit, the
thread (8), warp and tile (4096) boundaries, negative keys and values, chunked
pushes.  Integer results are bit-exact and the output is in key order."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C2 = ("count", "sum", "min", "max")


def _run(keys, vals, aggs, chunks=1):
    from oracle import oracle as O
    from paper_1311_0059_b200.core import AggSpec
    from paper_1311_0059_b200.engine import GroupBy
    agg = AggSpec.from_names(list(aggs))
    n = len(keys)
    with GroupBy("sort_based", agg, ["i64"], ["i64"], budget_groups=-1) as g:
        step = -(-n // chunks)
        for s in range(0, n, step):
            g.push([keys[s:s + step]], [vals[s:s + step]])
        res = g.result()
    assert res.sorted
    uk, want, _ = O.groupby_numpy([keys], [vals], O.ospec(list(aggs)))
    assert res.n_groups == len(uk)
    # emitted in key order (unsigned word order = the reference's byte order)
    assert np.array_equal(res.keys[0], uk[:, 0].view(np.int64))
    assert np.array_equal(res.as_float64(), want)


@pytest.mark.parametrize("aggs", [C2, ("count", "sum")])
def test_sort_near_unique_keys(aggs):
    rng = np.random.default_rng(1)
    keys = rng.integers(0, 1 << 40, 700_001).astype(np.int64)
    vals = rng.integers(-1000, 1000, len(keys)).astype(np.int64)
    _run(keys, vals, aggs, chunks=3)


def test_sort_long_segments():
    """A few keys hold most of the records (segments of 10^5 records: k_seg_long2),
    next to 100K keys seen once or twice."""
    rng = np.random.default_rng(2)
    hot = rng.choice(np.array([5, -7, 1 << 33], np.int64), 600_000)
    cold = rng.integers(-(1 << 20), 1 << 20, 150_000).astype(np.int64)
    keys = rng.permutation(np.concatenate([hot, cold]))
    vals = rng.integers(-(1 << 40), 1 << 40, len(keys)).astype(np.int64)
    _run(keys, vals, C2)


def test_sort_segment_lengths_around_the_boundaries():
    """Segments of every length around the thread's 8 records, the walk limit
    (256) and the tile (4096), laid end to end so they start at every offset."""
    rng = np.random.default_rng(3)
    lens = np.concatenate([np.arange(1, 20), [31, 32, 33, 63, 64, 65, 255, 256, 257, 258, 263, 264, 265, 511, 512,
                                              513, 4095, 4096, 4097, 8191, 8193], rng.integers(1, 300, 400)])
    lens = rng.permutation(lens)
    keys = np.repeat(np.arange(len(lens), dtype=np.int64) * 3 - 500, lens)
    vals = rng.integers(-5, 5, len(keys)).astype(np.int64)
    p = rng.permutation(len(keys))
    _run(keys[p], vals[p], C2)
    _run(keys[p], vals[p], ("count", "sum"), chunks=2)


def test_sort_single_key_and_tiny_inputs():
    rng = np.random.default_rng(4)
    _run(np.full(50_000, -3, np.int64), rng.integers(0, 9, 50_000).astype(np.int64), C2)
    _run(np.array([7], np.int64), np.array([1], np.int64), C2)
    _run(np.array([7, 7, 8, 9, 9, 9, 9, 9, 9, 9], np.int64), np.arange(10, dtype=np.int64), C2)
