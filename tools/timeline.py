"""Host-side phase timeline of one GroupBy run (reset / push / finish)."""
import argparse, os, sys, time
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
a = ap.parse_args()
cfg = D.CONFIGS[a.config]
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
for it in range(4):
    t0 = time.perf_counter(); g.reset(); s.synchronize(); t1 = time.perf_counter()
    g.push(keys, vals); s.synchronize(); t2 = time.perf_counter()
    g.finish(); s.synchronize(); t3 = time.perf_counter()
    print(f"run {it}: reset {1e3*(t1-t0):.3f} ms  push {1e3*(t2-t1):.3f} ms  finish {1e3*(t3-t2):.3f} ms", flush=True)
