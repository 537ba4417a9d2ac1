"""Planning of the hybrid operators, restated (hybrid.py:64-163, run_store.py:222-246).

Same names, arguments and results as the reference functions so code and
tests written against ``aggbench.operators`` work unchanged; the CUDA engine
(csrc/aggb200.cu ``plan``) applies the same rules to size its resident table
and uses Formula 1 as the floor of its spill fan-out.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from paper_1311_0059_b200.core import (DatasetStats, FIELD_SIZE, InvalidBudget, KLEN_SIZE,
                                       LINK_SIZE, MergeOrderError, SLOT_SIZE)

RECURSE = "recurse"
FALLBACK_HASH_SORT = "fallback_hash_sort"
HASH_SPACE = 1 << 32
BLOOM_BYTE = 1


@dataclass
class HybridHashPlan:
    """Partitioning decision for one hybrid-hash level (hybrid.py:68-86)."""

    M: int
    P: int
    F: float
    r_res: float
    r_spill: float
    grace_levels: int = 0
    P_s: float | None = None
    fallback_flags: tuple = ()
    _gf: float = field(default=0.0, repr=False)

    @property
    def group_frames(self) -> float:
        return self._gf


def plan_table(n_frames: int, frame_size: int, group_bytes: float, slot_ratio: float = 1.0,
               bloom: bool = False) -> tuple:
    """(capacity hint, n_slots) of a table in n_frames (hash_table.py:31-45)."""
    from paper_1311_0059_b200.core import CapacityExceeded
    if n_frames < 2:
        raise CapacityExceeded(f"table needs at least 2 frames, got {n_frames}")
    per_group = group_bytes + LINK_SIZE + slot_ratio * (SLOT_SIZE + (BLOOM_BYTE if bloom else 0))
    cap = int(n_frames * frame_size / per_group)
    return cap, max(1, math.ceil(slot_ratio * cap))


def fudge_factor(group_bytes: float, extra: float, slot_ratio: float = 1.0,
                 bloom: bool = False) -> float:
    per_group = group_bytes + LINK_SIZE + slot_ratio * (SLOT_SIZE + (BLOOM_BYTE if bloom else 0))
    return per_group * extra / max(group_bytes, 1e-300)


def plan_partitions(group_frames: float, M: int) -> int:
    """Formula 1: 0 in memory, else ceil((G*F - M) / (M - 2)) clamped to [1, M-2]."""
    if M < 3:
        raise InvalidBudget(f"partition planning needs M >= 3, got {M}")
    if group_frames <= M:
        return 0
    return max(1, min(math.ceil((group_frames - M) / (M - 2)), M - 2))


def plan_hybrid(stats: DatasetStats, M: int, F: float) -> HybridHashPlan:
    """P, the resident share and grace levels (grace iff G*F >= M^2)."""
    if M < 4:
        raise InvalidBudget(f"hybrid hashing needs M >= 4, got {M}")
    gf = stats.G * F
    levels = 0
    need = gf
    while need >= float(M) * M:
        levels += 1
        need = gf / float(M - 1) ** levels
    P = plan_partitions(gf, M)
    if P == 0:
        r_res, r_spill = 1.0, 0.0
    else:
        r_res = (M - P) / ((M - P) + M * P)
        r_spill = (1.0 - r_res) / P
    return HybridHashPlan(M=M, P=P, F=F, r_res=r_res, r_spill=r_spill, grace_levels=levels,
                          _gf=gf)


def plan_merge_rounds(n_runs: int, fan_in: int) -> list:
    """Algorithm-1 merge schedule (run_store.py:222-246)."""
    if fan_in < 2:
        raise MergeOrderError(f"fan-in must be >= 2, got {fan_in}")
    if n_runs == 0:
        return []
    if n_runs == 1:
        return [[0]]
    from collections import deque
    queue, rounds, nxt = deque(range(n_runs)), [], n_runs
    while len(queue) > fan_in:
        z = fan_in if len(queue) > 2 * fan_in - 1 else len(queue) - fan_in + 1
        rounds.append([queue.popleft() for _ in range(z)])
        queue.append(nxt)
        nxt += 1
    rounds.append(list(queue))
    return rounds


def merge_round_count(n_runs: int, fan_in: int) -> int:
    """len(plan_merge_rounds(n_runs, fan_in)) without building the schedule."""
    if n_runs <= 1:
        return n_runs
    q, rounds = n_runs, 0
    while q > fan_in:
        if q > 2 * fan_in - 1:
            k = (q - (2 * fan_in - 1) + fan_in - 2) // (fan_in - 1)  # full-width rounds in a batch
            k = max(1, k)
            q -= k * (fan_in - 1)
            rounds += k
        else:
            q -= q - fan_in
            rounds += 1
    return rounds + 1


def sort_merge_levels(input_frames: float, M: int) -> int:
    fan = max(2, M - 1)
    runs = max(1, math.ceil(input_frames / fan))
    return merge_round_count(runs, fan)


def fallback_controller(run_frames: float, parent_frames: float, level: int,
                        sort_levels: int) -> str:
    """Recurse, or fall back to hash-sort (80% / level rule)."""
    if parent_frames > 0 and run_frames > 0.8 * parent_frames:
        return FALLBACK_HASH_SORT
    if level > sort_levels:
        return FALLBACK_HASH_SORT
    return RECURSE


def make_cuts(r_res: float, P: int) -> np.ndarray:
    """Ascending partition cutoffs over the 32-bit hash space."""
    if P == 0:
        return np.array([HASH_SPACE], np.int64)
    c0 = max(1, int(r_res * HASH_SPACE))
    rest = HASH_SPACE - c0
    cuts = np.array([c0] + [c0 + (rest * (i + 1)) // P for i in range(P)], np.int64)
    cuts[P] = HASH_SPACE
    return cuts


def dd_spill_trajectory(G_t: float, M: int, nparts: int, overhead: int,
                        groups_per_frame: float) -> list:
    """Expected dynamic-destaging evictions (hybrid.py:918-944)."""
    if nparts <= 0 or groups_per_frame <= 0:
        return []
    g_full = G_t / nparts
    cuts = []
    for s in range(nparts):
        residents = nparts - s
        g_cap = max((M - overhead - 1 - s), 0) * groups_per_frame
        if residents * g_full <= g_cap:
            break
        cuts.append(max(g_cap / residents, 0.0))
    return cuts


def predict_dd_spills(G_t: float, M: int, nparts: int, overhead: int,
                      groups_per_frame: float) -> int:
    return len(dd_spill_trajectory(G_t, M, nparts, overhead, groups_per_frame))


def group_bytes_for(stats: DatasetStats, frame_size: int, state_width: int) -> float:
    """Operator.group_bytes (base.py:141-147)."""
    if stats.G_t > 0 and stats.G > 0:
        return max(stats.G * frame_size / stats.G_t, KLEN_SIZE + 1 + FIELD_SIZE * state_width)
    return KLEN_SIZE + 16 + FIELD_SIZE * state_width
