import sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_1311_0059_b200 import datagen as D, engine as E
from paper_1311_0059_b200.core import AggSpec
cfg = D.scaled(D.CONFIGS["C2"], 600_000, key_range=60_000)
keys, vals = D.generate(cfg)
agg = AggSpec.from_names(list(cfg.aggs))
with E.GroupBy("pre_partitioning", agg, ["i64"], ["i64"], budget_groups=8000, emit_partials=True, seed=42) as g:
    g.push([keys[0][:300000]], [vals[0][:300000]])
    res = g.finish()
    buf, counts, rb = g.pack(2)
    rec = buf.cpu().numpy().view(np.int64).reshape(-1, rb // 8)[:res.n_groups]
    print('n', res.n_groups, 'counts', counts, 'unique packed keys', len(np.unique(rec[:, 0])), 'min/max', rec[:,0].min(), rec[:,0].max(), flush=True)
    print('last rows', rec[-3:].tolist())
    print('count col sum', rec[:, 1].sum(), 'records', 300000)
