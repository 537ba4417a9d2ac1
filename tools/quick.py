import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1311_0059_b200 import datagen as D, engine as E
from paper_1311_0059_b200.core import AggSpec
from oracle import oracle as O
cfg = D.scaled(D.CONFIGS['C2'], 2_000_000)
keys, vals = D.generate(cfg)
agg = AggSpec.from_names(list(cfg.aggs))
uk, out, _ = O.groupby_numpy(keys, vals, O.ospec(cfg.aggs))
for algo in ('pre_partitioning', 'original_hh', 'hash_sort'):
    for budget in (-1, 2500):
        t=time.time()
        try:
            with E.GroupBy(algo, agg, ['i64'], ['i64'], budget_groups=budget) as g:
                g.push(keys, vals)
                r = g.result().sorted_by_key()
                m = g.metrics()
            ok = r.n_groups == len(uk) and np.array_equal(r.keys[0], uk[:,0].view(np.int64)) and np.array_equal(r.as_float64(), out)
            print(algo, budget, 'groups', r.n_groups, len(uk), 'OK' if ok else 'MISMATCH', m['spilled_records'], m['recursion_depth'], m['kernel_launches'], '%.3fs'%(time.time()-t), flush=True)
        except Exception as e:
            print(algo, budget, 'ERR', type(e).__name__, e, flush=True)
