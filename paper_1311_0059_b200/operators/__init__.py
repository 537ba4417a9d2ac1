"""Aggregation operators behind one open / push / close interface.

Same registry and names as the reference (operators/__init__.py:37-120):
``OPERATORS[algo_id]``, ``ALGORITHM_IDS``, ``select_algorithm``, the planning
functions and ``run_operator`` / ``collect_groups``.  Every operator runs on
the B200 through libaggb200 (include/aggb200.h); the algorithm id selects the
GPU schedule:

* pre_partitioning — fill the L2-resident table, freeze it at a kernel
  boundary, probe (SMEM bloom first) and spill misses to HBM pages, recurse.
  For one-word keys, one int64 value and an integer COUNT/SUM/MIN/MAX spec:
  after the freeze every record is routed into the run of its hash range
  (k_scan_wc) and each run's compact child is seeded with the resident keys of
  that range, whose aggregates it merges into the table (csrc/wc2.cuh).
* original_hh — partition-0 table + raw spill of the other partitions,
  overflow cuts partition 0 into partial states (hybrid.py:431-451).
* hash_sort — aggregate until full, cut the table to a run of partial states,
  merge the runs with a fold (hash-partitioned children).
* sort_based — radix sort of the keys plus segmented reduction.
* shared_hash, dynamic_destaging — one table shared by every partition;
  records of a destaged partition spill raw (MODE_DD passes).  When the table
  runs dry, dynamic_destaging destages its largest resident partitions
  (hybrid.py:974-1149); shared_hash cuts every partition but partition 0 at the
  first overflow and partition 0 at the second (hybrid.py:579-915).
"""

from __future__ import annotations

from dataclasses import dataclass

from paper_1311_0059_b200.operators.base import (EngineConfig, FrameSource, OpContext, Operator,
                                                 collect_groups, run_operator)
from paper_1311_0059_b200.operators.planning import (FALLBACK_HASH_SORT, RECURSE, HybridHashPlan,
                                                     dd_spill_trajectory, fallback_controller,
                                                     fudge_factor, make_cuts, plan_hybrid,
                                                     plan_merge_rounds, plan_partitions, plan_table,
                                                     predict_dd_spills, sort_merge_levels)


class SortBased(Operator):
    algo_id = "sort_based"


class HashSort(Operator):
    algo_id = "hash_sort"


class OriginalHybridHash(Operator):
    algo_id = "original_hh"


class SharedHashing(Operator):
    algo_id = "shared_hash"


class DynamicDestaging(Operator):
    algo_id = "dynamic_destaging"


class PrePartitioning(Operator):
    algo_id = "pre_partitioning"


SORT_BASED = SortBased.algo_id
HASH_SORT = HashSort.algo_id
ORIGINAL_HH = OriginalHybridHash.algo_id
SHARED_HASH = SharedHashing.algo_id
DYNAMIC_DESTAGING = DynamicDestaging.algo_id
PRE_PARTITIONING = PrePartitioning.algo_id

OPERATORS = {cls.algo_id: cls for cls in (SortBased, HashSort, OriginalHybridHash,
                                           SharedHashing, DynamicDestaging, PrePartitioning)}
ALGORITHM_IDS = tuple(OPERATORS)


@dataclass
class SelectorInput:
    """What the caller knows about the input (operators/__init__.py:61-68)."""

    sorted: bool = False
    skewed: bool = False
    cardinality_confident: bool = True
    G_estimate: float = 0.0


def select_algorithm(s: SelectorInput) -> str:
    """Paper Fig. 17 decision (operators/__init__.py:71-84)."""
    if s.sorted:
        return SORT_BASED
    if s.skewed:
        return HASH_SORT
    return PRE_PARTITIONING


__all__ = ["ALGORITHM_IDS", "DYNAMIC_DESTAGING", "DynamicDestaging", "EngineConfig",
           "FALLBACK_HASH_SORT", "FrameSource", "HASH_SORT", "HashSort", "HybridHashPlan",
           "OPERATORS", "ORIGINAL_HH", "OpContext", "Operator", "OriginalHybridHash",
           "PRE_PARTITIONING", "PrePartitioning", "RECURSE", "SHARED_HASH", "SORT_BASED",
           "SelectorInput", "SharedHashing", "SortBased", "collect_groups",
           "dd_spill_trajectory", "fallback_controller", "fudge_factor", "make_cuts",
           "plan_hybrid", "plan_merge_rounds", "plan_partitions", "plan_table",
           "predict_dd_spills", "run_operator", "select_algorithm", "sort_merge_levels"]
