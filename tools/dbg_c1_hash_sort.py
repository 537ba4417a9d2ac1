"""Diagnostic: C1 hash_sort metrics and phase trace (AGGB_TRACE=1)."""
import sys
sys.path.insert(0, "/root/repo")
import torch, bench
from paper_1311_0059_b200 import datagen as D
from paper_1311_0059_b200.engine import GroupBy
from paper_1311_0059_b200.core import DatasetStats
cfg = D.CONFIGS["C1"]
keys, vals = bench.make_inputs(cfg, 0, cfg.n, torch.device("cuda", 0))
st = DatasetStats(R=1, R_t=cfg.n, G=1, G_t=min(cfg.key_range, cfg.n))
for algo in ("hash_sort", "pre_partitioning"):
    g = GroupBy(algo, bench.spec_of(cfg), bench.types_of(keys), bench.types_of(vals),
                budget_groups=bench.budget_of(cfg, cfg.n), stats=st, seed=1)
    g.push(keys, vals); r = g.finish(); print(algo, "groups", r.n_groups, g.metrics())
