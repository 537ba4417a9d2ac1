import sys, os
sys.path.insert(0, "/root/repo")
import torch, bench
from paper_1311_0059_b200 import datagen as D
from paper_1311_0059_b200.engine import GroupBy
from paper_1311_0059_b200.core import DatasetStats
cfg = D.scaled(D.CONFIGS["C5"], 10_000_000)
keys, vals = bench.make_inputs(cfg, 0, cfg.n, torch.device("cuda", 0))
st = DatasetStats(R=1, R_t=cfg.n, G=1, G_t=min(4194304, cfg.n))
g = GroupBy("hash_sort", bench.spec_of(cfg), bench.types_of(keys), bench.types_of(vals), budget_groups=cfg.budget_groups, stats=st, seed=1)
g.push(keys, vals); r = g.finish(); print("groups", r.n_groups, g.metrics())
