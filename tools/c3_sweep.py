"""C3 at every Zipf exponent (s = 0.5, 1.0, 1.5), 200M records: step time + check."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1311_0059_b200 import datagen as D
from paper_1311_0059_b200.engine import GroupBy
from paper_1311_0059_b200.core import DatasetStats

dev = torch.device("cuda", 0)
for s_ in (0.5, 1.0, 1.5):
    cfg = D.scaled(D.CONFIGS["C3"], D.CONFIGS["C3"].n, zipf_s=s_)
    keys, vals = bench.make_inputs(cfg, 0, cfg.n, dev)
    st = DatasetStats(R=1, R_t=cfg.n, G=1, G_t=min(cfg.zipf_k, cfg.n))
    for algo in ("pre_partitioning", "hash_sort"):
        s = torch.cuda.Stream()
        g = GroupBy(algo, bench.spec_of(cfg), bench.types_of(keys), bench.types_of(vals),
                    budget_groups=bench.budget_of(cfg, cfg.n), stats=st, seed=1234, stream=s)
        for it in range(3):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            g.reset(); e0.record(s); g.push(keys, vals); res = g.finish(); e1.record(s); torch.cuda.synchronize()
        kk, vv = g.result_torch()
        m = g.metrics()
        print(json.dumps({"cfg": "C3", "s": s_, "algo": algo, "ms": round(e0.elapsed_time(e1), 2),
                          "groups": res.n_groups, "count_ok": int(vv[0].sum().item()) == cfg.n,
                          "spilled": m["spilled_records"], "resident": m["resident_groups"]}), flush=True)
        g.close()
    del keys, vals
    torch.cuda.empty_cache()
