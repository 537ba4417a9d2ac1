"""Host-side logic that needs no GPU: the wire codec, key word encoding, the
spec surface, dataset-stat validation and the generator's determinism."""

import numpy as np
import pytest

from paper_1311_0059_b200 import core
from paper_1311_0059_b200 import datagen as D
from paper_1311_0059_b200.core import AggSpec, DatasetStats, SpecError
from paper_1311_0059_b200.operators.base import decode_keys, encode_frames, encode_keys


def test_pack_fixed_matches_frames_from_records():
    rng = np.random.default_rng(1)
    kb = rng.integers(0, 256, (777, 8), dtype=np.uint8)
    kb[:, 0] |= 1
    st = rng.random((777, 3))
    ref = core.frames_from_records([(kb[i].tobytes(), st[i].tolist()) for i in range(777)], 3, 1024)
    mine = core.pack_fixed(kb, st, 1024)
    assert len(ref) == len(mine)
    assert all(np.array_equal(a, b) for a, b in zip(ref, mine))
    keys, vals = core.unpack_fixed(mine, 3)
    assert np.array_equal(keys, kb) and np.array_equal(vals, st)


def test_unpack_detects_variable_keys():
    fr = core.frames_from_records([(b"k1", [1.0]), (b"k22", [2.0])], 1, 256)
    assert core.unpack_fixed(fr, 1) is None
    assert list(core.iter_records(fr[0], 1)) == [(b"k1", (1.0,)), (b"k22", (2.0,))]


def test_key_words_are_injective_and_order_preserving():
    keys = [b"k1", b"k1\x00", b"k10", b"k2", b"\x00", b"\xff" * 15, b"a" * 15, b"ab", b"b"]
    words = []
    for k in keys:
        a, b = encode_keys(np.frombuffer(k, np.uint8)[None, :], len(k))
        words.append((int(a[0]) & (2**64 - 1), int(b[0]) & (2**64 - 1)))
        assert decode_keys(a, b) == [k]
    assert len(set(words)) == len(keys)
    # unsigned word order == the reference's byte order (_kernels.py:121-131)
    assert [k for _, k in sorted(zip(words, keys))] == sorted(keys)


def test_encode_frames_round_trip_variable_lengths():
    keys = [b"a", b"bbbb", b"cc"]
    vals = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    frames = list(encode_frames(keys, vals, 64))
    got = [r for fr in frames for r in core.iter_records(fr, 2)]
    assert got == [(k, tuple(v)) for k, v in zip(keys, vals.tolist())]


def test_spec_surface():
    s = AggSpec.from_names("count,sum,avg")
    assert s.state_width == 4 and s.out_width == 3
    assert list(s.finish_src) == [0, 1, 2]
    assert s.finish(s.merge(s.init(3.0), s.init(5.0))) == (2.0, 8.0, 4.0)
    with pytest.raises(SpecError):
        AggSpec.from_names("median")
    with pytest.raises(SpecError):
        AggSpec.from_names(["sum"], bind=(0, 1))


def test_dataset_stats_validation():
    with pytest.raises(SpecError):
        DatasetStats(R=1, R_t=10, G=1, G_t=11)
    DatasetStats(R=1, R_t=10, G=1, G_t=10)


def test_generator_is_deterministic_and_sliceable():
    cfg = D.scaled(D.CONFIGS["C2"], 10_000)
    k1, v1 = D.generate(cfg)
    k2, v2 = D.generate(cfg, 4_000, 3_000)
    assert np.array_equal(k1[0][4_000:7_000], k2[0]) and np.array_equal(v1[0][4_000:7_000], v2[0])
    assert k1[0].min() >= 0 and k1[0].max() < cfg.key_range
    cfg5 = D.scaled(D.CONFIGS["C5"], 1000)
    keys, vals = D.generate(cfg5)
    assert keys[1].dtype == np.int32 and len(vals) == 4
    rows = D.wide_rows(keys, vals)
    assert rows.shape == (1000, 64)
    assert np.array_equal(rows[:, 16:24].copy().view(np.int64)[:, 0], vals[0])


def test_zipf_generator_shape():
    cfg = D.scaled(D.CONFIGS["C3"], 100_000, zipf_s=1.5)
    keys, _ = D.generate(cfg)
    _, counts = np.unique(keys[0], return_counts=True)
    assert counts.max() > 0.3 * len(keys[0])  # s = 1.5: the top key takes ~38%


def test_choose_exchange_rule():
    """partial groups when local aggregation shrinks the bytes
    to send, raw rows otherwise (C2 partial at any N; C4 raw at 8 GPUs)."""
    from paper_1311_0059_b200.exchange import choose_exchange, expected_distinct
    assert abs(expected_distinct(1e9, 627_500_000) / 1e9 - 0.5) < 0.01  # C4: ~0.5N distinct
    assert choose_exchange(100_000_000, 1_000_000, 16, 40) == "partial"  # C2 per GPU
    assert choose_exchange(125_000_000, 627_500_000, 16, 24) == "raw"    # C4 at 8 GPUs
    assert choose_exchange(1_000_000, 10_000, 16, 24) == "partial"       # C1
    assert choose_exchange(0, 10, 16, 24) == "partial"


# measured on B200 (profiles/r02_all_configs_full.jsonl; C3 and C5 unchanged since r01), ms
_MEASURED = {
    "C2": (dict(n=1e8, groups=1e6, rec_bytes=16, state_bytes=40, out_bytes=40, budget_groups=125000,
                key_bits=20, compact=True), {"pre_partitioning": 1.61, "original_hh": 5.64, "shared_hash": 10.3,
                                             "dynamic_destaging": 16.1}),
    "C3s05": (dict(n=2e8, groups=1e7, state_bytes=24, out_bytes=32, key_bits=24),
              {"pre_partitioning": 9.09, "hash_sort": 26.7}),
    "C3s1": (dict(n=2e8, groups=8.9e6, state_bytes=24, out_bytes=32, key_bits=24, hot_share=0.16),
             {"pre_partitioning": 8.46, "hash_sort": 15.8}),
    "C4": (dict(n=1e9, groups=5e8, key_bits=30), {"sort_based": 68.4, "hash_sort": 356.6,
                                                  "pre_partitioning": 104.7}),
    "C5": (dict(n=5e8, groups=4194304, rec_bytes=64, state_bytes=120, out_bytes=144, budget_groups=83886,
                key_bits=44, spill_rec_bytes=48), {"pre_partitioning": 56.2, "hash_sort": 401.0}),
}


@pytest.mark.parametrize("cfg", sorted(_MEASURED))
def test_gpu_cost_model_orders_like_the_measurements(cfg):
    """the GPU byte/time model ranks the config's algorithms
    in the measured order and lands within 3x of every measured time (~25% for
    the streaming schedules)."""
    from paper_1311_0059_b200.operators.gpu_cost import Workload, model, select_algorithm_gpu
    kw, meas = _MEASURED[cfg]
    w = Workload(**kw)
    pred = {a: model(a, w).ms for a in meas}
    best_meas = min(meas, key=meas.get)
    assert min(pred, key=pred.get) == best_meas
    assert select_algorithm_gpu(w, algos=tuple(meas)) == best_meas
    for a, m in meas.items():
        assert m / 3 <= pred[a] <= 3 * m, (a, pred[a], m)
        if a in ("pre_partitioning", "original_hh", "sort_based"):
            assert abs(pred[a] - m) <= 0.3 * m, (a, pred[a], m)


def test_gpu_cost_model_bytes_follow_the_survey_formulas():
    """C2 pre-partitioning: 16 B read per record, the 7/8 spill written and re-read
    at 16 B, 40 B out per group (4.44 GB)."""
    from paper_1311_0059_b200.operators.gpu_cost import Workload, model
    r = model("pre_partitioning", Workload(1e8, 1e6, 16, 40, 40, 125000, 20))
    assert abs((r.bytes_read + r.bytes_written) / 1e9 - 4.44) < 0.01
    assert abs(r.spill_bytes / 1e9 - 1.4) < 0.01
