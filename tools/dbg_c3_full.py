"""Bisect the C3 full-size fp64 SUM mismatch (run under env overrides)."""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import bench
from paper_1311_0059_b200 import datagen as D
import test_gpu_fullsize as T

s = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
algo = sys.argv[2] if len(sys.argv) > 2 else "pre_partitioning"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 200_000_000
cfg = dataclasses.replace(D.CONFIGS["C3"], zipf_s=s)
if n != cfg.n:
    cfg = D.scaled(cfg, n)
dev = torch.device("cuda", 0)
keys, vals = bench.make_inputs(cfg, 0, cfg.n, dev)
rk, rv, met = T._run(algo, cfg, keys, vals)
ck = rk[0]; order = torch.argsort(ck); ck = ck[order]
uk, want, absum = T._reference(keys, vals, cfg)
print("env", {k: v for k, v in os.environ.items() if k.startswith("AGGB")}, "s", s, "n", cfg.n, algo)
print("groups", uk.numel(), ck.numel(), "metrics", {k: met[k] for k in ("spilled_records", "recursion_depth", "partitions_level0")})
same = uk.numel() == ck.numel() and torch.equal(uk, ck)
print("keys equal", same)
if same:
    cnt = want[0]
    got_c = rv[0][order]
    print("count equal", torch.equal(got_c, cnt))
    g = rv[1][order]; w = want[1]
    d = g - w
    bad = d.abs() > 1e-9 * absum[1]
    nb = int(bad.sum())
    print("bad sums", nb)
    if nb:
        idx = torch.nonzero(bad)[:, 0]
        print("bad count stats: min", int(cnt[idx].min()), "max", int(cnt[idx].max()), "median", float(cnt[idx].double().median()))
        print("all count median", float(cnt.double().median()))
        print("got>want frac", float((d[idx] > 0).double().mean()))
        r = d[idx] / (w[idx] / cnt[idx])  # in units of a mean value
        print("diff / mean value: ", r[:20].tolist())
        print("rank of bad keys (first 20 by count)", torch.sort(cnt[idx], descending=True)[0][:20].tolist())
