"""GPU parity at BASELINE.json's full sizes (C2 100M, C3 200M at s = 0.5/1/1.5,
C4 1B, C5 500M wide rows) for every algorithm the config names, against the
CPU oracle: the C port of the reference operators (oracle/aggoracle.c, pinned
to reference-run goldens by tests/test_oracle_golden.py), run over the very
same input bytes (copied from the device) in key-disjoint shards on the host's
cores (oracle/fullsize.py; one oracle run per config, shared by its algorithms).

Per group, after sorting by key: identical group sets; COUNT, integer
SUM/MIN/MAX (and AVG of integer columns) and fp64 MIN/MAX bit-exact; fp64
SUM/AVG within 1e-9 relative (BASELINE.json north_star), except where the
group's sum cancels (|sum| < 1e-4 x sum|x|, C5's normal(0,1) columns): there the
two summation orders (the reference's and the GPU's atomics) differ by up to
~n eps sum|x|, so such groups are held to 1e-12 x sum|x| (the summation-order
bound with margin) and counted.  The observed maximum relative and
sum|x|-scaled errors are printed (profiles/r02_fullsize_parity.jsonl).
Size-independent properties are checked too: unique output keys, sum of COUNT
= N, integer SUM totals and global MIN/MAX.

Inputs come from the device generator (bench.make_inputs), exactly as the
benchmark sees them.
"""

import json

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

REL = 1e-9  # fp64 SUM/AVG tolerance (BASELINE.json north_star)
CANCEL = 1e-4  # |sum| below this x sum|x|: a cancelling group (see the module docstring)
ABS_CANCEL = 1e-12  # their bound, x sum|x|

_ORACLE = {}  # config -> (key columns, values): one oracle run per config


def _oracle(cfg, keys, vals):
    """The C port over the same bytes (cached per config across algorithms)."""
    import dataclasses
    import numpy as np
    from oracle import fullsize as F
    tag = (cfg.name, cfg.n, cfg.zipf_s)
    if tag not in _ORACLE:
        _ORACLE.clear()  # one full-size config in host memory at a time
        hk = [k.cpu().numpy() for k in keys]
        hv = [v.cpu().numpy() for v in vals]
        G = cfg.key_range or cfg.zipf_k or cfg.k0_range * cfg.k1_range
        _ORACLE[tag] = F.port_groupby(hk, hv, cfg.aggs, cfg.bind, groups=min(G, cfg.n)) + (hk, hv)
        del hk, hv
    return _ORACLE[tag]


def _exact_sum(hk, hv, key, b):
    """math.fsum of one group's values (the correctly rounded sum)."""
    import math
    import numpy as np
    m = hk[0] == key[0]
    for i in range(1, len(hk)):
        m &= hk[i] == key[i]
    return math.fsum(np.asarray(hv[b])[m].tolist()), int(m.sum())


def _composite(keys):
    import torch
    if len(keys) == 1:
        return keys[0]
    # C5: k0 int64 in [0, 4096), k1 int32 in [0, 1024): order-preserving packing
    return keys[0] * (1 << 32) + keys[1].to(torch.int64)


def _reference_absum(keys, vals, cfg):
    """Per-group sum of |x| of the float columns (the summation-order scale),
    by sorting on the device (test-only)."""
    import torch
    kk = _composite(keys)
    uk, inv = torch.unique(kk, sorted=True, return_inverse=True)
    G = uk.numel()
    cnt = torch.bincount(inv, minlength=G)
    cols, absum = [], []
    for name, b in zip(cfg.aggs, cfg.bind):
        v = vals[b]
        isf = v.dtype == torch.float64
        if name == "count":
            cols.append(cnt.clone())
            absum.append(None)
        elif name in ("sum", "avg"):
            s = torch.zeros(G, dtype=v.dtype, device=v.device).index_add_(0, inv, v)
            a = torch.zeros(G, dtype=torch.float64, device=v.device).index_add_(0, inv, v.abs()) if isf else None
            if name == "avg":
                s = s.to(torch.float64) / cnt.to(torch.float64)
                a = a / cnt.to(torch.float64) if isf else None
            cols.append(s)
            absum.append(a)
        else:
            red = "amin" if name == "min" else "amax"
            o = torch.zeros(G, dtype=v.dtype, device=v.device).scatter_reduce_(0, inv, v, red, include_self=False)
            cols.append(o)
            absum.append(None)
    return uk, cols, absum


def _run(algo, cfg, keys, vals):
    import torch
    import bench
    from paper_1311_0059_b200.core import DatasetStats
    from paper_1311_0059_b200.engine import GroupBy
    G = cfg.key_range or cfg.zipf_k or cfg.k0_range * cfg.k1_range
    st = DatasetStats(R=1, R_t=cfg.n, G=1, G_t=min(G, cfg.n))
    with GroupBy(algo, bench.spec_of(cfg), bench.types_of(keys), bench.types_of(vals),
                 budget_groups=bench.budget_of(cfg, cfg.n), stats=st, seed=1234) as g:
        g.push(keys, vals)
        g.finish()
        rk, rv = g.result_torch()
        met = g.metrics()
    torch.cuda.synchronize()
    return rk, rv, met


def _check(cfg, algo):
    import torch
    import bench
    from paper_1311_0059_b200 import datagen as D
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    keys, vals = bench.make_inputs(cfg, 0, cfg.n, dev)
    rk, rv, met = _run(algo, cfg, keys, vals)
    n_out = rk[0].numel()
    # properties
    ck = _composite(rk)
    order = torch.argsort(ck)
    ck = ck[order]
    assert n_out == 0 or bool((ck[1:] > ck[:-1]).all()), "duplicate output keys"
    ci = list(cfg.aggs).index("count")
    assert int(rv[ci].sum().item()) == cfg.n, "sum of COUNT != N"
    for j, (name, b) in enumerate(zip(cfg.aggs, cfg.bind)):
        v = vals[b]
        if v.dtype == torch.float64:
            continue
        if name == "sum":
            assert int(rv[j].sum().item()) == int(v.sum().item()), (name, b)
        elif name == "min":
            assert rv[j].min().item() == v.min().item()
        elif name == "max":
            assert rv[j].max().item() == v.max().item()
    # per group against the oracle (the C port over the same bytes)
    import numpy as np
    ok_keys, ok_vals, hk, hv = _oracle(cfg, keys, vals)
    assert len(ok_keys[0]) == n_out, (len(ok_keys[0]), n_out)
    got_keys = [k[order].cpu().numpy().astype(np.int64) for k in rk]
    for a, b in zip(got_keys, ok_keys):
        assert np.array_equal(a, b), "group keys differ from the oracle"
    del rk
    _, _, absum = _reference_absum(keys, vals, cfg)
    stats = {"config": cfg.name, "algorithm": algo, "zipf_s": cfg.zipf_s, "groups": int(n_out)}
    for j, name in enumerate(cfg.aggs):
        got = rv[j][order].to(torch.float64).cpu().numpy()
        want = ok_vals[:, j]
        if absum[j] is None:
            assert np.array_equal(got, want), (j, name, np.flatnonzero(got != want)[:5])
            continue
        ax = absum[j].cpu().numpy()
        d = np.abs(got - want)
        rel = d / np.maximum(np.abs(want), 1e-300)
        cancel = np.abs(want) < CANCEL * ax
        bad_rel = (rel > REL) & ~cancel
        bad_abs = cancel & (d > ABS_CANCEL * ax)
        stats[f"{name}[{cfg.bind[j]}]"] = {"max_rel": float(rel[~cancel].max()) if (~cancel).any() else 0.0,
                                          "max_rel_all_groups": float(rel.max()),
                                          "groups_over_1e-9_rel": int((rel > REL).sum()),
                                          "max_abs_over_sum_abs": float((d / np.maximum(ax, 1e-300)).max()),
                                          "cancelling_groups": int(cancel.sum())}
        assert not bad_rel.any(), (j, name, int(bad_rel.sum()), float(rel[~cancel].max()))
        assert not bad_abs.any(), (j, name, int(bad_abs.sum()))
        # groups past 1e-9 relative (cancelling sums): against the correctly rounded
        # sum, the GPU's error is of the same order as the reference's own
        if name == "sum":
            off = []
            for g in np.flatnonzero(rel > REL)[:8]:
                ex, cnt = _exact_sum(hk, hv, [k[g] for k in ok_keys], cfg.bind[j])
                e_gpu, e_ref = abs(got[g] - ex), abs(want[g] - ex)
                off.append({"records": cnt, "exact": ex, "gpu": float(got[g]), "reference": float(want[g]),
                            "gpu_err_over_sum_abs": e_gpu / ax[g], "ref_err_over_sum_abs": e_ref / ax[g]})
                assert e_gpu <= 1e-12 * ax[g] and e_ref <= 1e-12 * ax[g]
            stats[f"{name}[{cfg.bind[j]}]"]["past_1e-9_rel"] = off
    print("PARITY " + json.dumps(stats))
    return met


CASES = [("C2", "pre_partitioning", {}), ("C2", "original_hh", {}), ("C2", "shared_hash", {}),
         ("C2", "dynamic_destaging", {}),
         ("C3", "pre_partitioning", {"zipf_s": 0.5}), ("C3", "pre_partitioning", {"zipf_s": 1.0}),
         ("C3", "pre_partitioning", {"zipf_s": 1.5}), ("C3", "hash_sort", {"zipf_s": 0.5}),
         ("C3", "hash_sort", {"zipf_s": 1.0}), ("C3", "hash_sort", {"zipf_s": 1.5}),
         ("C4", "sort_based", {}), ("C4", "hash_sort", {}),
         ("C5", "pre_partitioning", {}), ("C5", "hash_sort", {})]


@pytest.mark.parametrize("name,algo,over", CASES, ids=[f"{c}-{a}-{o.get('zipf_s', '')}" for c, a, o in CASES])
def test_full_size(name, algo, over):
    import dataclasses
    import torch
    from paper_1311_0059_b200 import datagen as D
    cfg = dataclasses.replace(D.CONFIGS[name], **over)
    try:
        met = _check(cfg, algo)
    finally:
        torch.cuda.empty_cache()
    if cfg.budget_groups:
        assert met["spilled_records"] > 0  # the budget forces spill at full size
