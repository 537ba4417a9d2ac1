"""Randomised runs of budgeted pre_partitioning over one-word keys and one int64
value (the write-combined level 0: k_scan_wc / k_child2_wc, and its fallback)
against the numpy oracle.    python tools/fuzz_wc.py [iterations] [seed]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(rng, it):
    from oracle import oracle as O
    from paper_1311_0059_b200.core import AggSpec, DatasetStats
    from paper_1311_0059_b200.engine import GroupBy
    n = int(rng.choice([3_000, 40_000, 300_000, 1_500_000]))
    G = int(rng.choice([7, 300, 5_000, 60_000, 400_000]))
    G = min(G, n)
    kind = rng.choice(["uniform", "sorted", "hot", "zipf", "runs"])
    base = rng.integers(0, G, n)
    if kind == "sorted":
        base = np.sort(base)
    elif kind == "hot":
        base = np.where(rng.random(n) < 0.7, rng.integers(0, 3, n), base)
    elif kind == "zipf":
        base = np.minimum(rng.zipf(1.3, n) - 1, G - 1)
    elif kind == "runs":
        base = np.repeat(rng.integers(0, G, n // 50 + 1), 50)[:n]
    kw = rng.choice(["small", "u32", "wide", "neg"])
    if kw == "small":
        keys = base.astype(np.int64)
    elif kw == "u32":
        keys = (base.astype(np.int64) * 7919 + 0xFFFFFF00) & 0xFFFFFFFF
    elif kw == "wide":
        keys = base.astype(np.int64) * 6_000_000_007 + (1 << 40)
    else:
        keys = -base.astype(np.int64) * 104_729 - 1
    if rng.random() < 0.1:
        keys[rng.integers(0, n, 5)] = np.iinfo(np.int64).min  # the sentinel key
    vw = rng.choice(["small", "i32", "i64"])
    if vw == "small":
        vals = rng.integers(-50, 1000, n)
    elif vw == "i32":
        vals = rng.integers(-(1 << 31), 1 << 31, n)
    else:
        vals = rng.integers(-(1 << 62), 1 << 62, n)
    keys = keys.astype(np.int64)
    vals = vals.astype(np.int64)
    aggs = ("count", "sum", "min", "max") if rng.random() < 0.7 else ("count", "sum")
    distinct = len(np.unique(keys))
    budget = int(max(2, distinct * rng.choice([0.01, 0.125, 0.5, 0.9])))
    G_t = int(min(n, max(1, distinct * rng.choice([1.0, 1.0, 0.2, 3.0]))))
    chunks = int(rng.choice([1, 1, 2, 5, 9]))
    agg = AggSpec.from_names(list(aggs))
    st = DatasetStats(R=1, R_t=n, G=1, G_t=G_t)
    with GroupBy("pre_partitioning", agg, ["i64"], ["i64"], budget_groups=budget, stats=st,
                 seed=int(rng.integers(1, 1 << 30))) as g:
        step = -(-n // chunks)
        for s in range(0, n, step):
            g.push([keys[s:s + step]], [vals[s:s + step]])
        res = g.result().sorted_by_key()
        met = g.metrics()
    uk, want, _ = O.groupby_numpy([keys], [vals], O.ospec(list(aggs)))
    tag = (it, n, G, kind, kw, vw, aggs, budget, G_t, chunks)
    assert res.n_groups == len(uk), (tag, res.n_groups, len(uk))
    assert np.array_equal(res.keys[0], uk[:, 0].view(np.int64)), tag
    got = res.as_float64()
    assert np.array_equal(got, want), (tag, np.argwhere(got != want)[:3])
    assert met["records"] == n and 0 <= met["spilled_records"] <= n, (tag, met)
    return tag


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    for it in range(iters):
        tag = one(rng, it)
        if it % 20 == 0:
            print("ok", tag, flush=True)
    print("fuzz ok:", iters, "cases")


if __name__ == "__main__":
    main()
