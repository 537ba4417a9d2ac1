"""Benchmark: input records/sec aggregated + HBM-roofline fraction (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--algo pre_partitioning]
    python bench.py --impl reference ...      # the reference's CPU path (oracle port)

Workload (N=1): BASELINE.json configs[1] = C2 — 100M records of (int64 key,
int64 value), keys uniform over 1M values, COUNT/SUM/MIN/MAX, resident-table
budget of 1/8 of the groups (125,000), pre-partitioning (hybrid-hash numbers
are reported beside it).  Inputs come from the seeded counter-based generator
(paper_1311_0059_b200/datagen.py, run on the device) and stay resident in HBM;
1.6 GB of input exceeds the 126 MB L2, so no L2 flush is needed between steps.

Under torchrun (N>1) every rank aggregates its own N-record shard (weak
scaling) and the partial groups are hash-exchanged with one NCCL all-to-allv
(torch.distributed) and merged; the step time is the max over ranks of the
device time (CUDA events on the engine's stream).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "input records/sec aggregated and % of HBM-bandwidth roofline at 1/2/4/8 B200"


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        import threading
        self.lines = []
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
            return self
        self.first = threading.Event()

        def reader():
            for ln in self.p.stdout:
                if ln.strip():
                    self.lines.append(ln)
                    self.first.set()
        self.t = threading.Thread(target=reader, daemon=True)
        self.t.start()
        return self

    def wait_sampling(self, timeout=5.0):
        """Block until the sampler is up (NVML initialised), so its start-up
        does not overlap the timed region."""
        if self.p is not None:
            self.first.wait(timeout)

    def __exit__(self, *exc):
        if self.p is not None:
            time.sleep(0.15)
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                pass
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_inputs(cfg, start, n, device):
    """Generate the shard [start, start+n) on the device (datagen.cu twin)."""
    import torch
    from paper_1311_0059_b200 import datagen as D
    from paper_1311_0059_b200 import _native as N
    L = N.load()
    st = torch.cuda.current_stream().cuda_stream

    def gen(kind, stream_id, lo=0, rng=1, dtype=torch.int64, cdf=None, K=0, a=0, b=0, out=None,
            stride=0):
        out = torch.empty(n, dtype=dtype, device=device) if out is None else out
        N.check(L.aggb_generate(st, kind, cfg.seed, stream_id, start, n, lo, rng,
                                cdf.data_ptr() if cdf is not None else None, K, a, b,
                                out.data_ptr(), stride), "aggb_generate")
        return out

    if cfg.wide:
        # C5: 64-byte rows  k0 i64 | k1 i32 | pad | v0 v1 i64 | v2 v3 f64 | pad (datagen.wide_rows)
        rows = torch.zeros((n, 64), dtype=torch.uint8, device=device)

        def field(off, dt):
            w = torch.tensor([], dtype=dt).element_size()
            return rows[:, off:off + w].view(dt)[:, 0]

        k0, k1 = field(0, torch.int64), field(8, torch.int32)
        v = [field(16, torch.int64), field(24, torch.int64), field(32, torch.float64),
             field(40, torch.float64)]
        gen(0, D.S_KEY, 0, cfg.k0_range, out=k0, stride=64)
        gen(4, D.S_K1, 0, cfg.k1_range, out=k1, stride=64)
        gen(0, D.S_V0, 0, 1 << 20, out=v[0], stride=64)
        gen(0, D.S_V1, 0, 1 << 20, out=v[1], stride=64)
        gen(2, D.S_V2, out=v[2], stride=64)
        gen(2, D.S_V3, out=v[3], stride=64)
        make_inputs.rows = rows
        return [k0, k1], v
    if cfg.zipf_k:
        cdf = torch.from_numpy(D.zipf_cdf(cfg.zipf_k, cfg.zipf_s)).to(device)
        a, b = D.zipf_perm_params(cfg.zipf_k, cfg.seed)
        keys = [gen(3, D.S_KEY, cdf=cdf, K=cfg.zipf_k, a=a, b=b)]
    else:
        keys = [gen(0, D.S_KEY, 0, cfg.key_range)]
    if cfg.value == "u01":
        vals = [gen(1, D.S_VAL, dtype=torch.float64)]
    else:
        vals = [gen(0, D.S_VAL, 0, 1000)]
    return keys, vals


def rec_bytes(cfg):
    kb = 12 if cfg.wide else 8
    vb = 32 if cfg.wide else 8
    return kb, vb


def spec_of(cfg):
    from paper_1311_0059_b200.core import AggSpec
    return AggSpec.from_names(list(cfg.aggs), bind=list(cfg.bind))


def types_of(cols):
    import torch
    return ["i64" if c.dtype == torch.int64 else "i32" if c.dtype == torch.int32 else "f64"
            for c in cols]


def budget_of(cfg, n_total):
    return cfg.budget_groups if cfg.budget_groups else -1


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args, rank, world, device):
    import torch
    from paper_1311_0059_b200 import datagen as D
    from paper_1311_0059_b200.engine import GroupBy
    from paper_1311_0059_b200.core import DatasetStats

    cfg = D.CONFIGS[args.config]
    if args.records:
        cfg = D.scaled(cfg, args.records)
    n = cfg.n
    keys, vals = make_inputs(cfg, rank * n, n, device)
    torch.cuda.synchronize()
    kb, vb = rec_bytes(cfg)
    G_est = (cfg.key_range or cfg.zipf_k or cfg.k0_range * cfg.k1_range)
    stats = DatasetStats(R=n * (kb + vb) / 32768, R_t=n, G=min(G_est, n) * 40 / 32768,
                         G_t=min(G_est, n))
    stream = torch.cuda.Stream(device=device)
    agg = spec_of(cfg)
    # N > 1: exchange partial groups after a local combine, or raw rows first
    # when the combine would not shrink what is sent
    xmode = None
    meta = None
    if world > 1:
        from paper_1311_0059_b200.exchange import choose_exchange
        meta = torch.distributed.new_group(backend="gloo")  # host-side counts exchange (no device sync)
        n_cols = len(keys) + len(vals)
        part_b = 8 * (len(keys) + len(spec_of(cfg).fns) + 1)  # key words + states (upper bound)
        xmode = args.exchange if args.exchange != "auto" else choose_exchange(n, G_est, 8 * n_cols, part_b)
    g = GroupBy(args.algo, agg, types_of(keys), types_of(vals), budget_groups=budget_of(cfg, n),
                stats=stats, seed=1234, device=device.index, stream=stream,
                emit_partials=xmode == "partial")
    xg = xr = None
    if xmode == "partial":
        from paper_1311_0059_b200.exchange import Exchanger
        xg = Exchanger(g, agg, types_of(keys), types_of(vals), device, stream, rank, world, meta_group=meta,
                       expect_groups=min(G_est, n * world) / world,
                       stats=stats, seed=1234, budget_groups=budget_of(cfg, n))
    elif xmode == "raw":
        from paper_1311_0059_b200.exchange import RawExchanger
        xr = RawExchanger(g, device, stream, meta_group=meta)

    def step():
        if xr is not None:
            xr.run(keys, vals)
            return
        g.reset()
        g.push(keys, vals)
        g.finish()
        if xg is not None:
            xg.run()

    clk = Clocks(device.index)
    with clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        clk.wait_sampling()
        launches = 0
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
            launches += g.metrics()["kernel_launches"]
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ms = e0.elapsed_time(e1) / args.steps
        # per-kernel durations: the same K steps again with a CUDA event pair around
        # every launch (kept out of the region above: the event records and their
        # collection add ~0.4 ms per step)
        g.profile(True)
        for _ in range(args.steps):
            step()
        ks = g.kernel_stats()
        g.profile(False)
    met = g.metrics()
    res_groups = met["output_groups"]
    if xg is not None or xr is not None:
        res_groups = (xg.merge if xg is not None else g).metrics()["output_groups"]
        t = torch.tensor([res_groups], dtype=torch.int64, device=device)
        torch.distributed.all_reduce(t)
        res_groups = int(t.item())
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    out = dict(ms=ms, kernels=ks, metrics=met, launches=launches, clocks=clk.summary(),
               n=n, cfg=cfg, groups=res_groups, xmode=xmode)

    # e2e through the C ABI with pinned host buffers (H2D + D2H inside the timed
    # region); at N > 1 every rank pushes its shard from host memory, the
    # exchange and merge run inside the step, and the time is the max over ranks
    if not args.no_e2e:
        hk = [k.cpu().pin_memory() for k in keys]
        hv = [v.cpu().pin_memory() for v in vals]
        ge = GroupBy(args.algo, agg, types_of(keys), types_of(vals),
                     budget_groups=budget_of(cfg, n), stats=stats, seed=1234,
                     device=device.index, stream=stream, emit_partials=xmode == "partial")
        xe = xre = None
        if xmode == "partial":
            from paper_1311_0059_b200.exchange import Exchanger
            xe = Exchanger(ge, agg, types_of(keys), types_of(vals), device, stream, rank, world, meta_group=meta,
                           expect_groups=min(G_est, n * world) / world,
                           stats=stats, seed=1234, budget_groups=budget_of(cfg, n))
        elif xmode == "raw":
            from paper_1311_0059_b200.exchange import RawExchanger
            xre = RawExchanger(ge, device, stream, meta_group=meta)
        outk = outv = None

        def estep():
            nonlocal outk, outv
            hres = ge
            if xre is not None:  # raw-first: the shard goes to the device, then to its ranks
                with torch.cuda.stream(stream):
                    dk = [k.to(device, non_blocking=True) for k in hk]
                    dv = [v.to(device, non_blocking=True) for v in hv]
                res = xre.run(dk, dv)
            else:
                ge.reset()
                ge.push([k.numpy() for k in hk], [v.numpy() for v in hv])
                res = ge.finish()
            if xe is not None:
                res = xe.run()
                hres = xe.merge
            gn = res.n_groups
            if outk is None or outk[0].numel() < gn:
                outk = [torch.empty(max(gn, 1), dtype=k.dtype).pin_memory() for k in keys]
                outv = [torch.empty(max(gn, 1), dtype=torch.float64).pin_memory()
                        for _ in agg.fns]
            import ctypes
            from paper_1311_0059_b200 import _native as N
            kp = (ctypes.c_void_p * N.MAX_KEYS)(*[t.data_ptr() for t in outk])
            vp = (ctypes.c_void_p * N.MAX_FNS)(*[t.data_ptr() for t in outv])
            N.check(hres.L.aggb_copy_result(hres.h, kp, vp), "aggb_copy_result")
            return gn

        for _ in range(max(1, min(args.warmup, 2))):
            estep()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        ng = 0
        for _ in range(args.steps):
            ng = estep()
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / args.steps
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t.item())
        out["e2e"] = {"value": n * world / (ems / 1e3), "unit": "records/s",
                      "h2d_bytes_per_step": int(sum(k.numel() * k.element_size() for k in hk)
                                                + sum(v.numel() * v.element_size() for v in hv)),
                      "d2h_bytes_per_step": int(ng * (sum(k.element_size() for k in keys)
                                                      + 8 * len(agg.fns))),
                      "ms_per_step": ems,
                      "path": "aggb_push(on_host=1, pinned) -> aggb_finish -> aggb_copy_result"
                              + (" (+ exchange and merge per rank; h2d/d2h bytes are rank 0's)"
                                 if world > 1 else "")}
        if xe is not None:
            xe.merge.close()
        ge.close()
    g.close()
    return out


def roofline(out, args, peak):
    """Algorithmic bytes per launch of the dominant kernel / its event time."""
    cfg = out["cfg"]
    met = out["metrics"]
    ks = out["kernels"]
    n = out["n"]
    kb, vb = rec_bytes(cfg)
    in_b = kb + vb
    kw = 2 if cfg.wide else 1
    spill_rec = 8 * (kw + (4 if cfg.wide else 1))
    nout = len(cfg.aggs)
    out_b = 8 * kw + 8 * nout
    S = met["spilled_records"]
    G = met["output_groups"]
    R = met["resident_groups"]
    steps = args.steps
    groups = {}
    # level-0 pass (FILL + PROBE / ROUTE): reads the batch, writes the spill
    l0 = [k for k in ks if (k.startswith("k_pass<") and "GRACE" not in k) or k == "k_scan_wc"]
    if l0:
        ms = sum(ks[k][1] for k in l0) / steps
        nl = sum(ks[k][0] for k in l0) / steps
        groups["level0_pass"] = (ms, nl, in_b * n + spill_rec * S)
    ch = [k for k in ("k_child", "k_child_wc", "k_wc_build") if k in ks]
    if ch:
        ms = sum(ks[k][1] for k in ch) / steps
        nl = sum(ks[k][0] for k in ch) / steps
        groups["child_aggregate"] = (ms, nl, spill_rec * S + out_b * max(G - R, 0))
    if not groups:
        return None, {}
    table = {}
    for name, (ms, nl, b) in groups.items():
        table[name] = {"ms_per_step": round(ms, 4), "launches_per_step": nl,
                       "alg_bytes_per_step": int(b),
                       "achieved_gbs": round(b / (ms * 1e-3) / 1e9, 1) if ms > 0 else None}
    dom = max(groups, key=lambda k: groups[k][0])
    ms, nl, b = groups[dom]
    ach = b / (ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{args.config}:{args.algo}:{dom}")
    except Exception:
        pass
    return ({"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak[0],
             "unit": "GB/s", "frac": round(ach / peak[0], 4), "traffic": traffic,
             "alg_bytes_per_launch": int(b / max(nl, 1)), "peak_source": peak[1]}, table)


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (C restatement of the reference operators)
# ---------------------------------------------------------------------------


_SAMPLES = {}


def cpu_sample_run(cfg, algo, sample, threads):
    from oracle import oracle as O
    from paper_1311_0059_b200 import datagen as D
    key = (cfg.name, algo, sample, threads)
    if key not in _SAMPLES:  # generated, sharded and packed once (untimed), reused by every step
        keys, vals = D.generate(cfg, 0, sample)
        budget = cfg.budget_groups if cfg.budget_groups else 1 << 40
        _SAMPLES[key] = O.prepare_port(algo if algo in O.ALGO_IDS else "pre_partitioning",
                                       keys, vals, cfg.aggs, cfg.bind, budget, threads=threads)
    dt, groups, met = O.run_prepared(_SAMPLES[key])
    return dt, groups


def cpu_baseline(cfg, algo, sample, threads):
    dt, groups = cpu_sample_run(cfg, algo, sample, threads)
    return {"value": round(sample / dt, 1), "unit": "records/s", "cores": threads,
            "kind": "port",
            "sample": f"first {sample:,} records of {cfg.name} (same generator, same group budget "
                      f"ratio, {threads} key-hash shards of the oracle port of {algo}); "
                      f"frame packing excluded", "seconds": round(dt, 3)}


def run_reference(args, rank, world):
    from paper_1311_0059_b200 import datagen as D
    cfg = D.CONFIGS[args.config]
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = args.cpu_sample
    vals = []
    for _ in range(args.warmup):
        cpu_sample_run(cfg, args.algo, min(sample, 200_000), threads)
    for _ in range(args.steps):
        dt, _ = cpu_sample_run(cfg, args.algo, sample, threads)
        vals.append(sample / dt)
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": "records/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sample / v * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "int64" if cfg.value != "u01" else "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "algorithm": args.algo, "records_per_gpu": cfg.n,
                       "global_records": cfg.n * world, "aggregates": list(cfg.aggs),
                       "key_universe": cfg.key_range or cfg.zipf_k or cfg.k0_range * cfg.k1_range,
                       "budget_groups": cfg.budget_groups or "in-memory",
                       "parallelism": "host cores of rank 0",
                       "records_per_step": sample, "note": "bounded sample of the workload"},
            "cpu_baseline": {"value": round(v, 1), "unit": "records/s", "cores": threads,
                             "kind": "port",
                             "sample": f"first {sample:,} records of {cfg.name} per step"},
            "e2e": {"value": round(v, 1), "unit": "records/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--algo", default="pre_partitioning")
    ap.add_argument("--records", type=int, default=0, help="records per GPU (default: config N)")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="auto", choices=("auto", "partial", "raw"),
                    help="N > 1: partial groups after a local combine, or raw rows first")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=50_000_000)
    ap.add_argument("--also", default="original_hh,shared_hash,dynamic_destaging",
                    help="extra algorithms to time (comma list)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # rank/channel/NVLS lines for the driver's check
        torch.distributed.init_process_group("nccl", device_id=device)
    out = run_ours(args, rank, world, device)
    extra = {}
    if rank == 0 and world == 1 and args.also:
        for algo in [a for a in args.also.split(",") if a and a != args.algo]:
            a2 = argparse.Namespace(**vars(args))
            a2.algo = algo
            a2.no_e2e = True
            o2 = run_ours(a2, rank, world, device)
            extra[algo] = {"value": round(o2["n"] * world / (o2["ms"] / 1e3), 1),
                           "ms_per_step": round(o2["ms"], 4),
                           "spilled_records": o2["metrics"]["spilled_records"]}
    if rank == 0:
        cfg = out["cfg"]
        n = out["n"]
        peak = peaks()
        roof, table = roofline(out, args, peak)
        value = n * world / (out["ms"] / 1e3)
        kb, vb = rec_bytes(cfg)
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "records/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(out["ms"], 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64" if cfg.value != "u01" else "f64",
            "data": "synthetic (seeded counter-based generator, datagen.py, generated on device)",
            "config": {"workload": cfg.name, "algorithm": args.algo, "records_per_gpu": n,
                       "global_records": n * world, "aggregates": list(cfg.aggs),
                       "key_universe": cfg.key_range or cfg.zipf_k or cfg.k0_range * cfg.k1_range,
                       "budget_groups": cfg.budget_groups or "in-memory",
                       "groups_out": out["groups"],
                       "l2": f"inputs {n * (kb + vb) / 1e9:.2f} GB/GPU > 126 MB L2; no flush",
                       "parallelism": f"dp{world} (shard + hash exchange of {out.get('xmode')} records)"
                       if world > 1 else "1 GPU"},
            "roofline": roof,
            "kernels": table,
            "gpu_launches": out["launches"],
            "clocks": out["clocks"],
            "metrics": {k: out["metrics"][k] for k in ("spilled_records", "resident_groups",
                                                        "spilled_partitions", "recursion_depth",
                                                        "partitions_level0", "budget_groups")},
        }
        if extra:
            line["other_algorithms"] = extra
        if "e2e" in out:
            line["e2e"] = out["e2e"]
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(cfg, args.algo, args.cpu_sample,
                                                os.cpu_count() or 1)
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
