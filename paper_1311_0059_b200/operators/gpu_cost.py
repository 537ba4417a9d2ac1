"""GPU byte/time cost model of the operators.

The reference's cost models (``aggbench/cost_models.py``: ``model_<algo>(stats,
params) -> CostReport``, frames of I/O and CPU work per algorithm) are
re-targeted here to the B200 path: every algorithm is a sequence of HBM
passes whose *algorithmic* bytes follow SURVEY.md §8(d) (input read, spill
written and re-read, sort passes, output), each pass priced at the fraction
of the measured HBM copy bandwidth its kernel reaches on B200
(profiles/r01_all_configs_full.jsonl, profiles/r01_notes.md), plus a random
sector term for in-memory tables larger than L2.  ``select_algorithm_gpu``
picks the cheapest algorithm; ``exchange_mode`` re-exports the raw-vs-partial
rule of the multi-GPU exchange.

The model is a planning aid, not a promise: it orders the algorithms like the
measurements on every BASELINE config (tests/test_host_logic.py), predicts the
streaming schedules (pre-partitioning, original hybrid hash, the sort path)
within ~25% on C2-C5, and the in-memory hash tables and hash_sort's cut loop
within ~3x (their random-access and launch costs are fitted, not derived).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from paper_1311_0059_b200.exchange import choose_exchange, expected_distinct

HBM_GBS = 6469.3         # MEASURED_PEAKS.json hbm_gbs (measured copy), B200
L2_BYTES = 126 << 20


@dataclass
class GpuCostParams:
    hbm_gbs: float = HBM_GBS
    l2_bytes: int = L2_BYTES
    # achieved fraction of the HBM roofline per pass kind (B200, session-3 profiles)
    eff: dict = field(default_factory=lambda: {
        "probe": 0.24,       # k_probe / k_probe_w: read input, write spill (C2 0.23, C3 0.26, C5 0.30)
        "child": 0.22,       # SMEM children: read spill (C2 0.23, C5 0.22)
        "scan_wc": 0.52,     # FILL + k_scan_wc (16-byte records, integer spec): C2 3.0 GB in 0.87 ms
        "child_wc": 0.39,    # k_wc2_build + k_child2_wc: C2 1.43 GB in 0.56 ms
        "split": 0.55,       # k_split: one more grace level over the spill
        "route": 0.11,       # k_pass ROUTE (original_hh): C2 4.25 ms for 3.0 GB
        "fill_l2": 0.20,     # table pass over an L2-resident table
        "radix": 0.40,       # one 8-bit one-sweep pass (C4: 32 GB in 12.3 ms), the append into the sort buffers
        "segreduce": 0.33,   # head counts + scan + the fused reduction (C4: 36 GB in 16.8 ms)
        "flush": 0.30,       # table compaction + finalize
    })
    rand_sector_ns: float = 0.095  # per random table sector beyond L2 (fit: C4 hash_sort FILL)
    split_fanout: int = 2200       # partitions one spill pass writes (k_probe SMEM)
    item_us: float = 0.07          # per child item (table init + flush), C4 fit
    destage_round_ms: float = 1.0  # dynamic_destaging: one destaging round (C2 fit)
    shared_stage_ms: float = 3.5   # shared_hash: one overflow stage (C2 fit)
    cut_us: float = 34.0           # hash_sort: one blind cut on the device (k_blind_cuts, C5: 5,960 cuts / 500M)


@dataclass
class GpuCostReport:
    algo: str
    bytes_read: float = 0.0
    bytes_written: float = 0.0
    spill_bytes: float = 0.0
    passes: list = field(default_factory=list)   # (kind, bytes, ms)

    @property
    def ms(self) -> float:
        return sum(p[2] for p in self.passes)

    def add(self, kind: str, rd: float, wr: float, pm: GpuCostParams, extra_ms: float = 0.0):
        self.bytes_read += rd
        self.bytes_written += wr
        ms = (rd + wr) / (pm.hbm_gbs * 1e9 * pm.eff[kind]) * 1e3 + extra_ms
        self.passes.append((kind, rd + wr, ms))


@dataclass
class Workload:
    """One aggregation: n records of rec_bytes (key + values), `groups` distinct
    keys, partial-state bytes per group, a budget in groups (0: in-memory)."""

    n: float
    groups: float
    rec_bytes: int = 16
    state_bytes: int = 24          # key + state words of a partial group
    out_bytes: int = 24            # key + finalized outputs
    budget_groups: float = 0.0
    key_bits: int = 64             # significant key bits (sort passes)
    spill_rec_bytes: int = 0       # raw spill record (0: rec_bytes; C5 rows 64 B -> 48 B)
    hot_share: float = 0.0         # share of records on heavy hitters (skew)
    compact: bool = False          # one-word key, one int64 value, integer COUNT/SUM/MIN/MAX: the
                                   # write-combined level 0 (k_scan_wc + k_child2_wc, csrc/wc2.cuh)

    @property
    def spill_bytes(self) -> int:
        return self.spill_rec_bytes or self.rec_bytes


def _spill_levels(spill_groups: float, child_groups: float, pm: GpuCostParams) -> int:
    need = max(1.0, spill_groups / max(1.0, 0.4 * child_groups))
    return 0 if need <= pm.split_fanout else 1


def _table_rand_ms(w: Workload, table_groups: float, pm: GpuCostParams) -> float:
    tbytes = table_groups * 2 * (w.state_bytes)
    miss = max(0.0, 1.0 - pm.l2_bytes / max(tbytes, 1.0))
    return w.n * (1.0 - w.hot_share) * miss * 3 * pm.rand_sector_ns * 1e-6


def model(algo: str, w: Workload, pm: GpuCostParams | None = None, child_groups: float = 1433) -> GpuCostReport:
    pm = pm or GpuCostParams()
    r = GpuCostReport(algo)
    inp = w.n * w.rec_bytes
    out = w.groups * w.out_bytes
    budget = w.budget_groups if w.budget_groups > 0 else math.inf
    if algo == "sort_based":
        passes = max(1, math.ceil(w.key_bits / 8))
        r.add("radix", inp, 0, pm)                       # load into the sort buffers
        for _ in range(passes):
            r.add("radix", inp, inp, pm)
        r.add("segreduce", inp + w.n * 8, out, pm)
        return r
    if algo == "hash_sort" and budget >= w.groups:
        r.add("fill_l2", inp, 0, pm, _table_rand_ms(w, w.groups, pm))
        r.add("flush", 0, out, pm)
        return r
    if algo == "hash_sort":
        # runs cut every `budget` distinct keys: partial states ~ records x collapse
        runs = w.n * min(1.0, expected_distinct(budget, w.groups) / budget if budget else 1.0)
        part = runs * w.state_bytes
        cuts = w.n / max(1.0, budget)  # one FILL + flush launch pair per cut (blind cuts)
        r.add("fill_l2", inp, part, pm, cuts * pm.cut_us * 1e-3)
        r.spill_bytes += part
        if _spill_levels(w.groups, child_groups, pm):
            r.add("split", 2 * part, part, pm)
        r.add("child", part, out, pm)
        return r
    # pre_partitioning / original_hh / the destaging schedules (same bytes; the
    # destaging ids add host-driven rounds: flush, per-partition histogram,
    # eviction, re-insert — fitted on C2: shared_hash 10.3 ms, dynamic_destaging 16 ms)
    extra = 0.0
    if algo == "dynamic_destaging" and w.groups > budget:
        extra = math.ceil(4 * math.log2(w.groups / budget + 1)) * pm.destage_round_ms
    elif algo == "shared_hash" and w.groups > budget:
        extra = 2 * pm.shared_stage_ms
    if algo == "pre_partitioning" and budget == math.inf and w.groups * 2 * w.state_bytes > 0.4 * pm.l2_bytes \
            and w.hot_share < 0.4:
        budget = 65536  # in-memory plans beyond L2 run at an L2-sized table (k_probe + bloom)
    resident = min(budget, w.groups)
    hit = 1.0 if resident >= w.groups else max(w.hot_share, resident / w.groups)
    if resident >= w.groups:
        r.add("fill_l2", inp, 0, pm, _table_rand_ms(w, w.groups, pm) if algo != "pre_partitioning" else 0.0)
        r.add("flush", 0, out, pm)
        return r
    spill = w.n * (1.0 - hit) * w.spill_bytes
    r.spill_bytes += spill
    if algo == "pre_partitioning" and w.compact and w.budget_groups > 0:
        # routing level 0 + seeded compact children (one wave pair, no split level);
        # the fixed term is the launch gaps and the closing round trip of a step
        r.add("scan_wc", inp, spill, pm)
        r.add("child_wc", spill, out - resident * w.out_bytes, pm, 0.13)
        return r
    r.add("route" if algo == "original_hh" else "probe", inp, spill, pm)
    if _spill_levels(w.groups - resident, child_groups, pm):
        r.add("split", 2 * spill, spill, pm)
    # children: one CTA per (sub-)partition; small items pay their table init and
    # flush (C4 pre-partitioning at 1B: 1.57M items of ~640 records, child 65 ms)
    items = max(1.0, (w.groups - resident) / (0.4 * child_groups))
    r.add("child", spill, out, pm, items * pm.item_us * 1e-3 + extra)
    return r


ALGOS = ("pre_partitioning", "original_hh", "shared_hash", "dynamic_destaging", "hash_sort", "sort_based")


def select_algorithm_gpu(w: Workload, pm: GpuCostParams | None = None, algos=ALGOS) -> str:
    """The algorithm with the lowest predicted time (ties: the order of ALGOS)."""
    return min(algos, key=lambda a: model(a, w, pm).ms)


def exchange_mode(w: Workload, n_gpus: int) -> str:
    """Raw vs partial exchange for an N-GPU run."""
    return choose_exchange(int(w.n / max(1, n_gpus)), w.groups, w.rec_bytes, w.state_bytes)
