"""Step time of the benchmark workload with/without kernel profiling (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1311_0059_b200 import datagen as D
from paper_1311_0059_b200.engine import GroupBy
from paper_1311_0059_b200.core import DatasetStats

cfg = D.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
dev = torch.device("cuda", 0)
keys, vals = bench.make_inputs(cfg, 0, cfg.n, dev)
n = cfg.n
kb, vb = bench.rec_bytes(cfg)
G_est = (cfg.key_range or cfg.zipf_k or cfg.k0_range * cfg.k1_range)
stats = DatasetStats(R=n * (kb + vb) / 32768, R_t=n, G=min(G_est, n) * 40 / 32768, G_t=min(G_est, n))
s = torch.cuda.Stream()
g = GroupBy("pre_partitioning", bench.spec_of(cfg), bench.types_of(keys), bench.types_of(vals),
            budget_groups=bench.budget_of(cfg, n), stats=stats, seed=1234, stream=s)
for prof in (False, True, False):
    for _ in range(3):
        g.reset(); g.push(keys, vals); g.finish()
    g.profile(prof)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(5):
        g.reset(); g.push(keys, vals); g.finish()
    e1.record(s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"profile={prof}: {e0.elapsed_time(e1)/5:.3f} ms/step (events)  {1e3*(t1-t0)/5:.3f} ms/step (wall)", flush=True)
