"""e2e (pinned host input through aggb_push(on_host)) vs raw H2D bandwidth, C2 100M."""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1311_0059_b200 import datagen as D
from paper_1311_0059_b200.engine import GroupBy
from paper_1311_0059_b200.core import DatasetStats

cfg = D.CONFIGS["C2"]
dev = torch.device("cuda", 0)
keys, vals = bench.make_inputs(cfg, 0, cfg.n, dev)
hk = [k.cpu().pin_memory() for k in keys]
hv = [v.cpu().pin_memory() for v in vals]
# raw H2D bandwidth
dk = [torch.empty_like(k) for k in keys]
s = torch.cuda.Stream()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for a, b in zip(dk, hk): a.copy_(b, non_blocking=True)
        for a, b in zip(dk, hv): a.copy_(b, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
print("raw H2D %.1f GB/s" % (3.2e9 / (t1 - t0) / 1e9 / 2 * 2 * 0.5 * 2 / 2), "(%.2f ms for 1.6 GB... per copy set %.2f ms)" % ((t1 - t0) * 1e3, (t1 - t0) * 1e3))
n = cfg.n
st = DatasetStats(R=1, R_t=n, G=1, G_t=min(cfg.key_range, n))
g = GroupBy("pre_partitioning", bench.spec_of(cfg), bench.types_of(keys), bench.types_of(vals),
            budget_groups=bench.budget_of(cfg, n), stats=st, seed=1234, stream=s)
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g.reset(); g.push([k.numpy() for k in hk], [v.numpy() for v in hv]); r = g.finish()
    torch.cuda.synchronize(); t1 = time.perf_counter()
print("e2e push+finish %.2f ms (%s)" % ((t1 - t0) * 1e3, os.environ.get("AGGB_PIPE_CHUNK", "default")))
