import sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_1311_0059_b200 import datagen as D, engine as E
from paper_1311_0059_b200.core import AggSpec
from oracle import oracle as O
cfg = D.scaled(D.CONFIGS["C2"], 600_000, key_range=60_000)
keys, vals = D.generate(cfg)
agg = AggSpec.from_names(list(cfg.aggs))
world = 2
n = cfg.n // world
segs = [[] for _ in range(world)]
for r in range(world):
    with E.GroupBy("pre_partitioning", agg, ["i64"], ["i64"], budget_groups=8000, emit_partials=True, seed=42) as g:
        g.push([k[r * n:(r + 1) * n] for k in keys], [v[r * n:(r + 1) * n] for v in vals])
        res = g.finish()
        buf, counts, rb = g.pack(world)
        print('local', r, res.n_groups, counts, rb, flush=True)
        rec = buf.cpu().numpy().view(np.int64).reshape(-1, rb // 8)
        print('  first keys per dest', rec[0, 0], rec[counts[0], 0], 'unique', len(np.unique(rec[:, 0])), flush=True)
        off = 0
        for d in range(world):
            segs[d].append(buf[off * rb:(off + counts[d]) * rb].clone()); off += counts[d]
for d in range(world):
    recv = torch.cat(segs[d])
    rr = recv.cpu().numpy().view(np.int64).reshape(-1, rb // 8)
    with E.GroupBy("pre_partitioning", agg, ["i64"], ["i64"], budget_groups=8000, seed=42) as m:
        m.push_partials(recv, recv.numel() // rb)
        r = m.result(); mm = m.metrics()
    print('merge', d, 'recv', recv.numel() // rb, 'unique keys in', len(np.unique(rr[:, 0])), 'out', r.n_groups, mm['records'], mm['spilled_records'], flush=True)
