"""C2-sized runs with skewed keys through the write-combined path (no cliff under skew)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1311_0059_b200.core import AggSpec, DatasetStats
from paper_1311_0059_b200.engine import GroupBy
n = 100_000_000
dev = torch.device("cuda", 0)
g0 = torch.Generator(device=dev); g0.manual_seed(1)
base = torch.randint(0, 1_000_000, (n,), device=dev, generator=g0, dtype=torch.int64)
vals = torch.randint(0, 1000, (n,), device=dev, generator=g0, dtype=torch.int64)
for name, keys in [("uniform", base),
                   ("30% on 3 keys", torch.where(torch.rand(n, device=dev, generator=g0) < 0.3, base % 3, base)),
                   ("sorted", torch.sort(base).values)]:
    agg = AggSpec.from_names(["count", "sum", "min", "max"])
    st = DatasetStats(R=1, R_t=n, G=1, G_t=1_000_000)
    s = torch.cuda.Stream()
    with GroupBy("pre_partitioning", agg, ["i64"], ["i64"], budget_groups=125_000, stats=st, seed=7, stream=s) as g:
        for it in range(2):
            if it == 1: g.profile(True)
            g.reset(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s); g.push([keys], [vals]); r = g.finish(); e1.record(s); torch.cuda.synchronize()
        print(name, "ms", round(e0.elapsed_time(e1), 2), "groups", r.n_groups, {k: round(v[1], 2) for k, v in g.kernel_stats().items()}, flush=True)
