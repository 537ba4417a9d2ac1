"""The reference's operator tests (test_operators.py) restated against the GPU
operators: frames of state records in, finished frames out, compared with a
dict oracle (conftest.py:23-139 pattern: quarter-integer values, string keys)."""

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GPU_ALGOS = ("pre_partitioning", "original_hh", "hash_sort", "shared_hash",
             "dynamic_destaging", "sort_based")


def build_dataset(n, m, seed, agg_names=("sum", "count"), dist="uniform", frame_size=1024,
                  key_style="short", sort_keys=False):
    from paper_1311_0059_b200.core import AggSpec, DatasetStats, frames_from_records
    agg = AggSpec.from_names(list(agg_names))
    rng = random.Random(seed)

    def mk_key(i):
        if key_style == "short":
            return f"k{i}".encode()
        return f"key-{i:08d}-{'x' * (i % 23)}".encode()

    recs, oracle = [], {}
    for j in range(n):
        if dist == "uniform":
            i = rng.randrange(m)
        elif dist == "hot":
            i = 0 if rng.random() < 0.6 else rng.randrange(m)
        elif dist == "single":
            i = 0
        else:
            i = (j * m) // max(n, 1)
        key = mk_key(i)
        val = rng.randrange(4000) / 4.0
        st = list(agg.init(val))
        recs.append((key, st))
        cur = oracle.get(key)
        oracle[key] = list(st) if cur is None else list(agg.merge(tuple(cur), tuple(st)))
    if sort_keys:
        recs.sort(key=lambda kv: kv[0])
    frames = frames_from_records(recs, agg.state_width, frame_size)
    m_true = len(oracle)
    rec_bytes = 2 + 8 + 8 * agg.state_width
    stats = DatasetStats(R=max(len(frames), 1), R_t=n,
                         G=(m_true * rec_bytes / frame_size) if n else 0.0, G_t=m_true)
    want = {k: list(agg.finish(tuple(st))) for k, st in oracle.items()}
    return frames, want, stats, agg


def drive(algo, frames, stats, agg, cfg, want=None):
    from paper_1311_0059_b200.core import iter_records
    from paper_1311_0059_b200.operators import OPERATORS, FrameSource, OpContext, run_operator
    with OpContext(cfg, agg) as ctx:
        op = OPERATORS[algo](ctx, stats)
        src = FrameSource.from_frames(frames, cfg.frame_size)
        got = {}
        for fr in run_operator(op, src):
            for k, vals in iter_records(fr, agg.out_width):
                assert k not in got, f"duplicate output key {k!r}"
                got[k] = list(vals)
        met = ctx.metrics
    if want is not None:
        assert set(got) == set(want)
        for k, v in want.items():
            assert got[k] == pytest.approx(v, abs=1e-9)
        assert met.output_groups == len(want)
    return got, met


@pytest.mark.parametrize("algo", GPU_ALGOS)
@pytest.mark.parametrize("n,m,M", [(60, 8, 8), (3000, 500, 6), (4000, 2500, 5)])
def test_operator_matches_oracle(algo, n, m, M):
    from paper_1311_0059_b200.operators import EngineConfig
    if algo == "dynamic_destaging" and M < 5:
        M = 5
    frames, want, stats, agg = build_dataset(n, m, seed=n + m + M,
                                             agg_names=("sum", "count", "min", "max"))
    drive(algo, frames, stats, agg, EngineConfig(memory_frames=M, frame_size=1024, seed=3), want)


@pytest.mark.parametrize("algo", GPU_ALGOS)
def test_long_keys_and_avg(algo):
    from paper_1311_0059_b200.operators import EngineConfig
    frames, want, stats, agg = build_dataset(3000, 700, seed=5, agg_names=("avg", "max", "sum"),
                                             key_style="long")
    drive(algo, frames, stats, agg, EngineConfig(memory_frames=8, frame_size=1024, seed=5), want)


@pytest.mark.parametrize("algo", GPU_ALGOS)
def test_empty_and_single_hot_key(algo):
    from paper_1311_0059_b200.operators import EngineConfig
    frames, want, stats, agg = build_dataset(0, 1, seed=1)
    got, met = drive(algo, frames, stats, agg, EngineConfig(memory_frames=8, frame_size=1024), want)
    assert got == {} and met.output_groups == 0
    frames, want, stats, agg = build_dataset(5000, 1, seed=2, dist="single", frame_size=512)
    got, _ = drive(algo, frames, stats, agg, EngineConfig(memory_frames=5, frame_size=512), want)
    assert len(got) == 1


@pytest.mark.parametrize("algo", GPU_ALGOS)
@pytest.mark.parametrize("wrong", [1.0, 1e7])
def test_misestimated_cardinality_stays_correct(algo, wrong):
    from paper_1311_0059_b200.operators import EngineConfig
    frames, want, stats, agg = build_dataset(3000, 900, seed=4)
    drive(algo, frames, stats, agg,
          EngineConfig(memory_frames=6, frame_size=1024, seed=4, group_estimate=wrong), want)


@pytest.mark.parametrize("algo,min_m", [("sort_based", 3), ("hash_sort", 3), ("original_hh", 4),
                                        ("shared_hash", 4),
                                        ("dynamic_destaging", 5), ("pre_partitioning", 4)])
def test_budget_floor(algo, min_m):
    from paper_1311_0059_b200.core import InvalidBudget
    from paper_1311_0059_b200.operators import EngineConfig
    frames, want, stats, agg = build_dataset(500, 120, seed=9)
    with pytest.raises(InvalidBudget):
        drive(algo, frames, stats, agg, EngineConfig(memory_frames=min_m - 1, frame_size=1024))
    drive(algo, frames, stats, agg, EngineConfig(memory_frames=min_m, frame_size=1024), want)


def test_sorted_input_streams_and_output_sorted():
    from paper_1311_0059_b200.operators import EngineConfig
    frames, want, stats, agg = build_dataset(3000, 700, seed=6, sort_keys=True)
    cfg = EngineConfig(memory_frames=4, frame_size=1024, seed=6, input_sorted=True)
    got, met = drive("sort_based", frames, stats, agg, cfg, want)
    assert list(got) == sorted(got)


def test_sorted_flag_rejects_unsorted_input():
    from paper_1311_0059_b200.core import MergeOrderError
    from paper_1311_0059_b200.operators import EngineConfig
    frames, _, stats, agg = build_dataset(2000, 500, seed=7)
    cfg = EngineConfig(memory_frames=4, frame_size=1024, seed=7, input_sorted=True)
    with pytest.raises(MergeOrderError):
        drive("sort_based", frames, stats, agg, cfg)


def test_sort_based_output_is_key_sorted_after_spill():
    from paper_1311_0059_b200.operators import EngineConfig
    frames, want, stats, agg = build_dataset(4000, 1500, seed=8)
    got, _ = drive("sort_based", frames, stats, agg,
                   EngineConfig(memory_frames=5, frame_size=1024, seed=8), want)
    assert list(got) == sorted(got)
