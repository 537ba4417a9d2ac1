"""Planning restated in paper_1311_0059_b200.operators.planning against known
answers produced by the reference itself (tests/golden/kat.json) and the
reference test suite's own examples (test_operators.py:47-79, :327-334)."""

import json
import os

import pytest

from conftest import GOLDEN_DIR
from paper_1311_0059_b200.core import DatasetStats, InvalidBudget
from paper_1311_0059_b200.operators import (FALLBACK_HASH_SORT, RECURSE, SelectorInput,
                                            fallback_controller, fudge_factor, make_cuts,
                                            plan_hybrid, plan_partitions, plan_table,
                                            select_algorithm, sort_merge_levels)

KAT = json.load(open(os.path.join(GOLDEN_DIR, "kat.json")))


def test_plan_partitions_kat():
    for g, m, want in KAT["plan_partitions"]:
        if m < 3:
            with pytest.raises(InvalidBudget):
                plan_partitions(g, m)
        else:
            assert plan_partitions(g, m) == want


def test_plan_hybrid_kat():
    for g, m, f, P, r_res, r_spill, levels in KAT["plan_hybrid"]:
        pl = plan_hybrid(DatasetStats(R=1e6, R_t=1e9, G=g, G_t=1e6), m, f)
        assert (pl.P, pl.grace_levels) == (P, levels)
        assert pl.r_res == pytest.approx(r_res, rel=1e-15)
        assert pl.r_spill == pytest.approx(r_spill, rel=1e-15, abs=1e-300)


def test_fudge_sort_levels_fallback_cuts_table_kat():
    for b, e, r, bl, want in KAT["fudge_factor"]:
        assert fudge_factor(b, e, r, bl) == pytest.approx(want, rel=1e-15)
    for f, m, want in KAT["sort_merge_levels"]:
        assert sort_merge_levels(f, m) == want
    for a, b, lv, sl, want in KAT["fallback"]:
        assert fallback_controller(a, b, lv, sl) == want
    for r, P, want in KAT["make_cuts"]:
        assert make_cuts(r, P).tolist() == want
    for nf, p, gb, sr, bl, want in KAT["plan_table"]:
        assert list(plan_table(nf, p, gb, sr, bl)) == want


def test_reference_examples():
    assert plan_partitions(1200.0, 100) == 12
    assert plan_partitions(1e9, 100) == 98
    stats = DatasetStats(R=1000, R_t=100000, G=150.0, G_t=10000)
    assert plan_hybrid(stats, 10, 1.0).grace_levels == 1
    assert plan_hybrid(stats, 13, 1.0).grace_levels == 0
    with pytest.raises(InvalidBudget):
        plan_hybrid(DatasetStats(R=10, R_t=100, G=5.0, G_t=50), 3, 1.2)
    assert fallback_controller(81, 100, 1, 5) == FALLBACK_HASH_SORT
    assert fallback_controller(10, 100, 5, 5) == RECURSE
    assert sort_merge_levels(100, 10) == 2


def test_select_algorithm_decision_table():
    assert select_algorithm(SelectorInput(sorted=True)) == "sort_based"
    assert select_algorithm(SelectorInput(sorted=True, skewed=True)) == "sort_based"
    assert select_algorithm(SelectorInput(skewed=True)) == "hash_sort"
    assert select_algorithm(SelectorInput()) == "pre_partitioning"
    assert select_algorithm(SelectorInput(cardinality_confident=False)) == "pre_partitioning"
