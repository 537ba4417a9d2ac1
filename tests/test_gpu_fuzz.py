"""Randomized drop-in cells against the GPU operators (the reference's
randomized operator fuzz, pkg/scratch_fuzz.py:24-132, restated): every cell
draws a frame size, a memory budget M, a record count, a key universe, an
aggregate list (with AVG), a key style (short / ~190-byte long / mixed), a key
distribution (uniform / hot / sorted runs) and a group-estimate mode (none,
exact, 64x under, 64x over), builds reference frames, and runs all six
operators through run_operator.  Each must: emit every group once (no
duplicate keys), leak no frames, keep its high-water mark within M, match a
dict oracle (values within 1e-9 + 1e-12 relative), and report output_groups.
A budget the operator rejects (InvalidBudget) skips that operator, as the
reference does.
"""

import random

import pytest

pytestmark = pytest.mark.gpu

ALGOS = ("sort_based", "hash_sort", "original_hh", "shared_hash", "dynamic_destaging", "pre_partitioning")
AGG_LISTS = (("sum",), ("count",), ("avg",), ("sum", "count", "min", "max"), ("min", "avg"),
             ("max", "sum", "avg"))


def _cell(seed):
    rng = random.Random(1000003 * seed + 17)
    return dict(fs=rng.choice([512, 1024, 4096]), M=rng.choice([4, 5, 6, 8, 12, 20, 40]),
                n=rng.choice([0, 1, 7, 100, 1000, 5000, 20000]),
                m=rng.choice([1, 2, 10, 100, 1000, 8000]), aggs=rng.choice(AGG_LISTS),
                keys=rng.choice(["short", "long", "mixed"]), dist=rng.choice(["uniform", "hot", "runs"]),
                est=rng.choice([None, "exact", "under", "over"]), rng=rng)


def _key(style, i):
    if style == "short":
        return b"k%d" % i
    if style == "long":  # ~190 bytes: dictionary-encoded on the host (keys > 15 bytes)
        return b"key-%09d-" % i + b"x" * 180
    return b"k%d" % i if i % 3 else b"key-%06d-" % i + b"y" * (i % 97)


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_cell(seed):
    from paper_1311_0059_b200.core import AggSpec, DatasetStats, InvalidBudget, frames_from_records, iter_records
    from paper_1311_0059_b200.operators import OPERATORS, EngineConfig, FrameSource, OpContext, run_operator
    c = _cell(seed)
    rng = c["rng"]
    n, m = c["n"], max(1, min(c["n"], c["m"]))
    agg = AggSpec.from_names(list(c["aggs"]))
    recs, states = [], {}
    for j in range(n):
        if c["dist"] == "uniform":
            i = rng.randrange(m)
        elif c["dist"] == "hot":
            i = 0 if rng.random() < 0.6 else rng.randrange(m)
        else:
            i = (j * m) // max(n, 1)
        k = _key(c["keys"], i)
        st = tuple(agg.init(rng.randrange(4000) / 4.0))
        recs.append((k, list(st)))
        states[k] = st if k not in states else agg.merge(states[k], st)
    want = {k: list(agg.finish(st)) for k, st in states.items()}
    fs = c["fs"]
    frames = frames_from_records(recs, agg.state_width, fs)
    g = len(want)
    gest = {None: None, "exact": float(max(g, 1)), "under": max(g / 64.0, 1.0), "over": g * 64.0 + 10}[c["est"]]
    rec_bytes = 2 + 8 + 8 * agg.state_width
    stats = DatasetStats(R=max(len(frames), 1), R_t=n, G=max(g * rec_bytes / fs, 1e-9) if n else 0.0, G_t=g)
    cfg = EngineConfig(memory_frames=c["M"], frame_size=fs, seed=seed, group_estimate=gest)
    ran = 0
    for algo in ALGOS:
        try:
            with OpContext(cfg, agg) as ctx:
                op = OPERATORS[algo](ctx, stats)
                got = {}
                for fr in run_operator(op, FrameSource.from_frames(frames, fs)):
                    for k, vals in iter_records(fr, agg.out_width):
                        assert k not in got, (algo, "duplicate key", k)
                        got[k] = list(vals)
                met, leaked = ctx.metrics, ctx.alloc.outstanding
        except InvalidBudget:
            continue
        assert leaked == 0, (algo, "leaked", leaked)
        assert met.high_water <= c["M"], (algo, "high water", met.high_water, c["M"])
        assert set(got) == set(want), (algo, len(set(want) - set(got)), len(set(got) - set(want)))
        for k, v in want.items():
            for a, b in zip(v, got[k]):
                assert abs(a - b) <= 1e-9 + 1e-12 * abs(a), (algo, k, v, got[k])
        assert met.output_groups == len(want), (algo, met.output_groups, len(want))
        ran += 1
    assert ran >= 1 or c["M"] < 5
