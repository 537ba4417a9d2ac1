"""Race stress (compute-sanitizer is closed on this pool, profiles/r02_notes.md):
the kernels that publish shared-memory state between threads without a
barrier in between (k_scan_wc's window word, ring, page maps and producer /
consumer flags; k_child2_wc's CAS inserts and idempotent flags; the generic drain's page maps and spin-free
claims) run many times over varied seeds, budgets, fan-outs and push
chunkings, and every run must equal the numpy oracle exactly (fp64 columns to
1e-9).  A lost or torn record, a duplicated group or a stale page shows up as a
mismatch."""

import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

CASES = [("C2", "pre_partitioning", 300_000, 4_000, {"key_range": 40_000}),
         ("C2", "pre_partitioning", 500_000, 1_500, {"key_range": 90_000}),
         ("C2", "original_hh", 300_000, 3_000, {"key_range": 30_000}),
         ("C2", "dynamic_destaging", 300_000, 3_000, {"key_range": 30_000}),
         ("C5", "pre_partitioning", 150_000, 2_000, {}),
         ("C2", "hash_sort", 300_000, 3_000, {"key_range": 30_000})]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("rep", range(3))
def test_repeated_runs_match_the_oracle(case, rep, monkeypatch):
    import sanitize_case
    name, algo, n, budget, over = CASES[case]
    if rep == 2:
        monkeypatch.setenv("AGGB_NO_WC", "1")  # the generic drain on the same input
    sanitize_case.run(name, algo, n + 7919 * rep, budget + 13 * rep, **over)
