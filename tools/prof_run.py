"""Profiling driver: one warm-up run + one run of a config, prints kernel stats.
Used as the <cmd> under ncu (see profiles/README.md)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1311_0059_b200 import datagen as D
from paper_1311_0059_b200.engine import GroupBy
from paper_1311_0059_b200.core import DatasetStats

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--algo", default="pre_partitioning")
ap.add_argument("--records", type=int, default=0)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--zipf-s", type=float, default=0.0)
a = ap.parse_args()
cfg = D.CONFIGS[a.config]
if a.zipf_s:
    import dataclasses
    cfg = dataclasses.replace(cfg, zipf_s=a.zipf_s)
if a.records:
    cfg = D.scaled(cfg, a.records)
dev = torch.device("cuda", 0)
keys, vals = bench.make_inputs(cfg, 0, cfg.n, dev)
torch.cuda.synchronize()
G = cfg.key_range or cfg.zipf_k or cfg.k0_range * cfg.k1_range
st = DatasetStats(R=1, R_t=cfg.n, G=1, G_t=min(G, cfg.n))
s = torch.cuda.Stream()
g = GroupBy(a.algo, bench.spec_of(cfg), bench.types_of(keys), bench.types_of(vals),
            budget_groups=bench.budget_of(cfg, cfg.n), stats=st, seed=1234, stream=s)
for r in range(a.runs):
    if r == a.runs - 1:
        g.profile(True)
    g.reset(); g.push(keys, vals); g.finish()
torch.cuda.synchronize()
print(json.dumps({"kernels": g.kernel_stats(), "metrics": g.metrics()}, indent=1))
