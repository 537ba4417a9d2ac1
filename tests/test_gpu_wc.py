"""The write-combined level 0 (csrc/wc2.cuh: k_scan_wc routes every record into
a spill partition or an owner run, k_child2_wc aggregates each run and merges
the owner runs' resident groups into the level-0 table) against the numpy
oracle, on the inputs that take its rare paths:

* runs that do not fit their child (tiny child tables, under-estimated
  cardinality): owner runs are gathered and re-probed by the
  generic PROBE, spill partitions go to the generic recursion;
* bursts (sorted input: a tile's records all claim one run, far past its ring
  window: held and parked records), chunked pushes (one chain of pages per CTA,
  run and launch), the sentinel key and the extreme keys, negative values and
  sums that need the wide (two-word) representation.

Integer results are bit-exact (BASELINE.json north_star)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(keys, vals, aggs, budget, chunks=1, G_t=None, seed=5):
    from oracle import oracle as O
    from paper_1311_0059_b200.core import AggSpec, DatasetStats
    from paper_1311_0059_b200.engine import GroupBy
    agg = AggSpec.from_names(list(aggs))
    n = len(keys)
    distinct = len(np.unique(keys))
    st = DatasetStats(R=1, R_t=n, G=1, G_t=G_t or distinct)
    with GroupBy("pre_partitioning", agg, ["i64"], ["i64"], budget_groups=budget, stats=st, seed=seed) as g:
        g.profile(True)
        step = -(-n // chunks)
        for s in range(0, n, step):
            g.push([keys[s:s + step]], [vals[s:s + step]])
        res = g.result().sorted_by_key()
        met = g.metrics()
        ks = g.kernel_stats()
    uk, want, _ = O.groupby_numpy([keys], [vals], O.ospec(list(aggs)))
    assert res.n_groups == len(uk) == distinct
    assert np.array_equal(res.keys[0], uk[:, 0].view(np.int64))
    got = res.as_float64()
    assert np.array_equal(got, want), np.argwhere(got != want)[:5]
    assert met["records"] == n
    return met, ks


C2 = ("count", "sum", "min", "max")


def _uniform(n, G, seed, lo=0, hi=1000):
    rng = np.random.default_rng(seed)
    return rng.integers(0, G, n).astype(np.int64), rng.integers(lo, hi, n).astype(np.int64)


def test_wc_path_runs_and_accounts_for_every_record():
    keys, vals = _uniform(600_000, 50_000, 1)
    met, ks = _run(keys, vals, C2, 6_000)
    assert "k_scan_wc" in ks and "k_child_wc" in ks and "k_child" not in ks
    # resident records were routed to owner runs but are not spilled records
    R = met["resident_groups"]
    assert 0.8 * 6_000 <= R <= 6_000
    assert 0 < met["spilled_records"] < 600_000
    assert met["spilled_records"] == met["level0_spilled_records"]


@pytest.mark.parametrize("aggs", [C2, ("count", "sum")])
@pytest.mark.parametrize("chunks", [1, 7])
def test_wc_chunked_pushes(aggs, chunks):
    keys, vals = _uniform(500_000, 30_000, 2 + chunks)
    _run(keys, vals, aggs, 3_000, chunks=chunks)


def test_wc_tiny_child_tables_fall_back(monkeypatch):
    """Every run overflows a 1 KB child table: owner runs are re-probed, spill
    partitions recurse through the generic drain."""
    monkeypatch.setenv("AGGB_WC_CHILD_KB", "1")
    keys, vals = _uniform(400_000, 40_000, 3)
    met, ks = _run(keys, vals, C2, 4_000)
    assert "k_scan_wc" in ks and "k_child" in ks
    assert 0 < met["spilled_records"] < 400_000


@pytest.mark.parametrize("aggs", [C2, ("count", "sum")])
def test_wc_values_beyond_int32(aggs):
    """Values beyond int32 take the children's 64-bit words (MIN/MAX as native 64-bit
    shared-memory atomics, sums with the value's high word), not the fallback."""
    rng = np.random.default_rng(4)
    keys = rng.integers(0, 20_000, 300_000).astype(np.int64)
    vals = rng.integers(-(1 << 45), 1 << 45, 300_000).astype(np.int64)
    met, ks = _run(keys, vals, aggs, 2_500)
    assert "k_scan_wc" in ks and "k_child" not in ks
    # the extremes, and 64-bit keys beside them
    vals[:8] = [np.iinfo(np.int64).max, np.iinfo(np.int64).min, -1, 0, 1 << 31, -(1 << 31) - 1, (1 << 32) + 5, 7]
    vals[8:16] = vals[:8][::-1]
    keys = keys * 6_000_000_007 - 17
    _run(keys, vals, aggs, 2_500)


def test_wc_underestimated_cardinality():
    """Ten times the groups the statistics promised: the runs hold more groups than
    their tables (fallback) or the output estimate; results are unaffected."""
    keys, vals = _uniform(800_000, 200_000, 5)
    _run(keys, vals, C2, 2_500, G_t=20_000)


def test_wc_sorted_input_bursts():
    """Sorted keys: long stretches of one key, so whole tiles claim one run (held
    records beyond the ring window, parked open-line records, several pages of a
    run opened in one tile)."""
    rng = np.random.default_rng(6)
    keys = np.sort(rng.integers(0, 3_000, 700_000)).astype(np.int64)
    vals = rng.integers(-500, 500, 700_000).astype(np.int64)
    _run(keys, vals, C2, 300)
    # and the reverse order (the resident keys are the largest ones)
    _run(keys[::-1].copy(), vals, C2, 300, chunks=3)


def test_wc_few_hot_spilled_keys():
    """Most records belong to a handful of keys that are NOT resident (they first
    appear after the table froze): one run takes most of every tile."""
    rng = np.random.default_rng(7)
    head = rng.permutation(5_000).astype(np.int64)            # fills the table (budget 500)
    hot = rng.integers(1_000_000, 1_000_004, 600_000).astype(np.int64)
    keys = np.concatenate([head, hot])
    vals = rng.integers(0, 100, len(keys)).astype(np.int64)
    _run(keys, vals, C2, 500)


def test_wc_sentinel_and_extreme_keys():
    rng = np.random.default_rng(8)
    pool = np.concatenate([np.array([np.iinfo(np.int64).min, np.iinfo(np.int64).max, -1, 0, 1,
                                     np.iinfo(np.int64).min + 1, 1 << 32, (1 << 32) + 1, -(1 << 32)], np.int64),
                           rng.integers(-(1 << 62), 1 << 62, 5_000)])
    keys = rng.choice(pool, 300_000)
    vals = rng.integers(-1000, 1000, 300_000).astype(np.int64)
    for budget in (4, 600):
        _run(keys, vals, C2, budget)
    # the sentinel key resident (first record) and spilled (first seen after the freeze)
    first = np.concatenate([[np.iinfo(np.int64).min], keys])
    _run(first, np.concatenate([[7], vals]), C2, 600)
    late = np.concatenate([keys[keys != np.iinfo(np.int64).min][:50_000], keys])
    _run(late, rng.integers(-1000, 1000, len(late)).astype(np.int64), C2, 600)


def test_wc_wide_sums():
    """Run sums beyond int32 (few groups, int32-sized values): the two-word sums."""
    rng = np.random.default_rng(9)
    keys = rng.integers(0, 3_000, 600_000).astype(np.int64)
    vals = rng.integers(-(1 << 30), 1 << 30, 600_000).astype(np.int64)
    _run(keys, vals, C2, 300)
    vals = rng.integers((1 << 30), (1 << 31) - 1, 600_000).astype(np.int64)
    _run(keys, vals, ("count", "sum"), 300)


def test_wc_keys_that_differ_in_the_high_word_only():
    rng = np.random.default_rng(10)
    keys = (rng.integers(0, 4_000, 400_000).astype(np.int64) << 32) | 5
    vals = rng.integers(0, 1000, 400_000).astype(np.int64)
    _run(keys, vals, C2, 400)


def test_wc_32bit_keys_and_their_escape_key():
    """Keys below 2^32 take the children's 32-bit tables; the key equal to their empty
    marker (0xFFFFFFFF) lives in the escape slot, resident or spilled."""
    rng = np.random.default_rng(11)
    pool = np.concatenate([np.array([0xFFFFFFFF, 0xFFFFFFFE, 0, 1, 0x80000000, 0x7FFFFFFF], np.int64),
                           rng.integers(0, 1 << 32, 6_000)])
    keys = rng.choice(pool, 400_000)
    vals = rng.integers(-1000, 1000, 400_000).astype(np.int64)
    _run(keys, vals, C2, 500)
    _run(np.concatenate([[0xFFFFFFFF], keys]).astype(np.int64), np.concatenate([[3], vals]), C2, 500)
    # one key beyond 32 bits, resident through FILL only (the runs stay 32-bit) and then also spilled
    _run(np.concatenate([[1 << 40], keys]).astype(np.int64), np.concatenate([[3], vals]), C2, 500)
    _run(np.concatenate([keys, [1 << 40]]).astype(np.int64), np.concatenate([vals, [3]]), C2, 500)


def test_wc_hot_run_overflows_its_page_list():
    """70% of the records on three keys: their runs take far more pages than the
    per-run lists hold (sized for the mean) and go on in the shared overflow list;
    no fallback is needed."""
    rng = np.random.default_rng(12)
    n = 3_000_000
    keys = np.where(rng.random(n) < 0.7, rng.integers(0, 3, n), rng.integers(0, 200_000, n)).astype(np.int64)
    vals = rng.integers(0, 1000, n).astype(np.int64)
    met, ks = _run(keys, vals, C2, 20_000, chunks=2)
    assert "k_scan_wc" in ks and "k_child" not in ks


@pytest.mark.parametrize("seed", [21, 22])
def test_wc_fuzz(seed):
    """Randomised shapes (tools/fuzz_wc.py): key distributions (uniform, sorted, hot,
    Zipf, runs), key widths, value widths, budgets, mis-estimated cardinalities, chunked
    pushes."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_wc
    rng = np.random.default_rng(seed)
    for it in range(40):
        fuzz_wc.one(rng, it)


def test_wc_heavy_hitters_are_reduced_in_the_scan():
    """A third of the records on three keys that are resident (seen first): every CTA
    finds them in its first tile and reduces their records per warp instead of routing
    them (their runs would otherwise take the whole step: 18.6 ms instead of 3.6 on C2);
    MIN/MAX and negative values included, and the same keys when they are NOT resident
    (first seen after the table froze) are routed like any other key."""
    rng = np.random.default_rng(13)
    n = 2_000_000
    base = rng.integers(0, 300_000, n)
    hot = np.array([7, -5, 1 << 41], np.int64)
    keys = np.where(rng.random(n) < 0.35, hot[rng.integers(0, 3, n)], base).astype(np.int64)
    vals = rng.integers(-(1 << 20), 1 << 20, n).astype(np.int64)
    met, ks = _run(keys, vals, C2, 30_000)
    assert "k_scan_wc" in ks and "k_child" not in ks
    assert met["spilled_records"] < 0.65 * n  # the hot keys' records are hits, not spills
    _run(keys, vals, ("count", "sum"), 30_000, chunks=3)
    # not resident: 40K other keys fill the table before the hot keys appear
    head = rng.permutation(40_000).astype(np.int64) + 1_000_000
    keys2 = np.concatenate([head, keys])
    vals2 = np.concatenate([rng.integers(0, 9, len(head)).astype(np.int64), vals])
    _run(keys2, vals2, C2, 30_000)
