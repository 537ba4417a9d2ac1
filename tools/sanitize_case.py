"""Small cases for compute-sanitizer (racecheck / synccheck): C2-shaped
pre_partitioning through the write-combined level 0 (k_scan_wc,
k_child2_wc) and through the generic drain (AGGB_NO_WC), C5-shaped wide rows,
hash_sort cuts.  Checked against the numpy oracle so a race that corrupts
results also fails here.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(name, algo, n, budget, **over):
    import torch
    import bench
    from oracle import oracle as O
    from paper_1311_0059_b200 import datagen as D
    from paper_1311_0059_b200.core import DatasetStats
    from paper_1311_0059_b200.engine import GroupBy
    cfg = D.scaled(D.CONFIGS[name], n, **over)
    dev = torch.device("cuda", 0)
    keys, vals = bench.make_inputs(cfg, 0, cfg.n, dev)
    torch.cuda.synchronize()
    G = cfg.key_range or cfg.k0_range * cfg.k1_range
    st = DatasetStats(R=1, R_t=cfg.n, G=1, G_t=min(G, cfg.n))
    with GroupBy(algo, bench.spec_of(cfg), bench.types_of(keys), bench.types_of(vals), budget_groups=budget,
                 stats=st, seed=3) as g:
        g.push(keys, vals)
        res = g.result().sorted_by_key()
    hk = [k.cpu().numpy() for k in keys]
    hv = [v.cpu().numpy() for v in vals]
    uk, want, _ = O.groupby_numpy(hk, hv, O.ospec(list(cfg.aggs)), list(cfg.bind))
    assert res.n_groups == len(uk), (name, algo, res.n_groups, len(uk))
    got = res.as_float64()
    fl = [i for i, (a, b) in enumerate(zip(cfg.aggs, cfg.bind)) if a in ("sum", "avg") and
          np.asarray(hv[b]).dtype.kind == "f"]
    for c in range(want.shape[1]):
        if c in fl:
            assert np.allclose(got[:, c], want[:, c], rtol=1e-9, atol=1e-9), (name, algo, c)
        else:
            assert np.array_equal(got[:, c], want[:, c]), (name, algo, c)
    print("ok", name, algo, res.n_groups)


if __name__ == "__main__":
    run("C2", "pre_partitioning", 300_000, 4_000, key_range=40_000)
    os.environ["AGGB_NO_WC"] = "1"
    run("C2", "pre_partitioning", 300_000, 4_000, key_range=40_000)
    del os.environ["AGGB_NO_WC"]
    run("C2", "original_hh", 200_000, 3_000, key_range=30_000)
    run("C5", "pre_partitioning", 100_000, 2_000)
    run("C2", "hash_sort", 200_000, 3_000, key_range=30_000)
