import sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_1311_0059_b200 import datagen as D, engine as E
from paper_1311_0059_b200.core import AggSpec
M=(1<<64)-1
def splitmix(z):
    z=(z+0x9E3779B97F4A7C15)&M; z=((z^(z>>30))*0xBF58476D1CE4E5B9)&M; z=((z^(z>>27))*0x94D049BB133111EB)&M; return z^(z>>31)
def fmix(k):
    k^=k>>33; k=(k*0xff51afd7ed558ccd)&M; k^=k>>33; k=(k*0xc4ceb9fe1a85ec53)&M; k^=k>>33; return k
cfg = D.scaled(D.CONFIGS["C2"], 600_000, key_range=60_000)
keys, vals = D.generate(cfg)
agg = AggSpec.from_names(list(cfg.aggs))
with E.GroupBy("pre_partitioning", agg, ["i64"], ["i64"], budget_groups=8000, emit_partials=True, seed=42) as g:
    g.push([keys[0][:300000]], [vals[0][:300000]])
    res = g.finish()
    for nr in (1, 2, 3, 4):
        buf, counts, rb = g.pack(nr)
        rec = buf.cpu().numpy().view(np.int64).reshape(-1, rb // 8)[:res.n_groups]
        seed = splitmix(splitmix(42) ^ 0x77)
        d = [((fmix(int(k) & M ^ seed) >> 32) * nr) >> 32 for k in rec[:2000, 0]]
        print(nr, counts, 'host dest of first 2000 packed:', np.bincount(d, minlength=nr).tolist(), 'keys', rec[:5, 0].tolist(), flush=True)
