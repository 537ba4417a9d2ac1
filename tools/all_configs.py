"""Run every BASELINE config once (after a warm-up) and print kernel times + checks."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1311_0059_b200 import datagen as D
from paper_1311_0059_b200.engine import GroupBy
from paper_1311_0059_b200.core import DatasetStats

# every config at its BASELINE.json size (C3 at each Zipf exponent); the
# AGGB_SCALED=1 environment keeps the older scaled C4 (200M) / C5 (100M) runs
FULL = not os.environ.get("AGGB_SCALED")
runs = [("C1", "pre_partitioning", 0, None), ("C1", "hash_sort", 0, None),
        ("C2", "pre_partitioning", 0, None), ("C2", "original_hh", 0, None),
        ("C2", "shared_hash", 0, None), ("C2", "dynamic_destaging", 0, None),
        ("C3", "pre_partitioning", 0, 0.5), ("C3", "pre_partitioning", 0, 1.0),
        ("C3", "pre_partitioning", 0, 1.5), ("C3", "hash_sort", 0, 0.5), ("C3", "hash_sort", 0, 1.0),
        ("C3", "hash_sort", 0, 1.5),
        ("C4", "sort_based", 0 if FULL else 200_000_000, None), ("C4", "hash_sort", 0 if FULL else 200_000_000, None),
        ("C5", "pre_partitioning", 0 if FULL else 100_000_000, None),
        ("C5", "hash_sort", 0 if FULL else 100_000_000, None)]
only = sys.argv[1:]
dev = torch.device("cuda", 0)
import dataclasses
for name, algo, nrec, zs in runs:
    if only and name not in only:
        continue
    cfg = D.CONFIGS[name]
    if zs is not None:
        cfg = dataclasses.replace(cfg, zipf_s=zs)
    if nrec:
        cfg = D.scaled(cfg, nrec)
    keys, vals = bench.make_inputs(cfg, 0, cfg.n, dev)
    torch.cuda.synchronize()
    G = cfg.key_range or cfg.zipf_k or cfg.k0_range * cfg.k1_range
    st = DatasetStats(R=1, R_t=cfg.n, G=1, G_t=min(G, cfg.n))
    s = torch.cuda.Stream()
    t0 = time.time()
    try:
        g = GroupBy(algo, bench.spec_of(cfg), bench.types_of(keys), bench.types_of(vals),
                    budget_groups=bench.budget_of(cfg, cfg.n), stats=st, seed=1234, stream=s)
        for it in range(2):
            if it == 1:
                g.profile(True)
            g.reset(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s); g.push(keys, vals); res = g.finish(); e1.record(s); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ks = {k: round(v[1], 2) for k, v in g.kernel_stats().items()}
        m = g.metrics()
        kk, vv = g.result_torch()
        cnt = vv[0].sum().item()  # COUNT column
        print(json.dumps({"cfg": name, "algo": algo, "s": zs, "n": cfg.n, "ms": round(ms, 2),
                          "Grec_s": round(cfg.n / ms / 1e6, 2), "groups": res.n_groups,
                          "count_sum_ok": int(cnt) == cfg.n, "spilled": m["spilled_records"],
                          "depth": m["recursion_depth"], "kernels": ks}), flush=True)
        g.close()
    except Exception as e:
        print(json.dumps({"cfg": name, "algo": algo, "error": f"{type(e).__name__}: {e}"}), flush=True)
    del keys, vals
    bench.make_inputs.rows = None  # C5's 64-byte rows (32 GB at full size)
    torch.cuda.empty_cache()
