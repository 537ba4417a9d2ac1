"""Dynamic destaging vs pre-partitioning on C2 shapes (diagnostic): results checked, step times."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1311_0059_b200 import datagen as D
from paper_1311_0059_b200.engine import GroupBy
from paper_1311_0059_b200.core import AggSpec, DatasetStats
from oracle import oracle as O
import time
for n, kr, bg in [(200_000, 20_000, 2500), (4_000_000, 40_000, 5000), (100_000_000, 1_000_000, 125_000)]:
    cfg = D.scaled(D.CONFIGS["C2"], n, key_range=kr)
    keys, vals = D.generate(cfg) if n <= 4_000_000 else (None, None)
    if keys is None:
        import bench
        dk, dv = bench.make_inputs(D.CONFIGS["C2"], 0, n, torch.device("cuda", 0))
    else:
        dk = [torch.from_numpy(k).cuda() for k in keys]; dv = [torch.from_numpy(v).cuda() for v in vals]
    agg = AggSpec.from_names(list(cfg.aggs))
    for algo in ("dynamic_destaging", "shared_hash", "pre_partitioning"):
        with GroupBy(algo, agg, ["i64"], ["i64"], budget_groups=bg, seed=3, stats=DatasetStats(R=1, R_t=n, G=1, G_t=kr)) as g:
            for it in range(2):
                g.reset(); torch.cuda.synchronize(); t0 = time.time()
                g.push(dk, dv); g.finish(); torch.cuda.synchronize(); ms = (time.time() - t0) * 1e3
            m = g.metrics()
            if keys is not None:
                res = g.result().sorted_by_key()
                uk, want, _ = O.groupby_numpy(keys, vals, O.ospec(cfg.aggs))
                ok = res.n_groups == len(uk) and np.array_equal(res.as_float64(), want)
            else:
                kk, vv = g.result_torch(); ok = int(vv[0].sum().item()) == n and kk[0].numel() == 1_000_000
            print(n, algo, f"{ms:.2f} ms", "ok" if ok else "MISMATCH", {k: m[k] for k in ("spilled_records", "spilled_partitions", "resident_groups", "recursion_depth")}, flush=True)
