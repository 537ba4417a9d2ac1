"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

For every config shape (scaled to sizes the reference finishes in seconds) and
every algorithm BASELINE.md times for it, the reference operator
(``OPERATORS[algo](ctx, stats)`` driven by ``run_operator``,
/root/reference/pkg/src/aggbench/operators/base.py:185-217) runs over frames
of the seeded inputs.  Output frames are decoded, sorted by key bytes and saved
with the reference's metrics.  The script also asserts that the vectorised
packer (oracle.pack_frames) is byte-identical to the reference's
``frames_from_records`` (core.py:251-265) and that all algorithms agree.

Fixtures hold (config, n, seed, generator knobs, input checksum, algorithm,
memory_frames, frame_size, engine seed, sorted keys, values, metrics) — never
the reference's source.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("AGGBENCH_TMP", tempfile.mkdtemp(prefix="golden-spill-"))

from aggbench.core import AggSpec, DatasetStats, frames_from_records  # noqa: E402
from aggbench.operators import OPERATORS, EngineConfig, OpContext, run_operator  # noqa: E402
from aggbench.run_store import FrameSource  # noqa: E402
from aggbench import _kernels as K  # noqa: E402

from oracle.oracle import init_states, ospec, pack_frames  # noqa: E402
from paper_1311_0059_b200 import datagen as D  # noqa: E402


def input_digest(keys, vals) -> str:
    h = hashlib.sha256()
    for a in list(keys) + list(vals):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def decode_fixed(frames_out, klen, width):
    rs = 2 + klen + 8 * width
    keys, vals = [], []
    for fr in frames_out:
        fr = np.asarray(fr, np.uint8)
        n = 0
        # fixed-width records: stop at the zero-length sentinel
        while (n + 1) * rs <= len(fr) and (fr[n * rs] | (fr[n * rs + 1] << 8)) != 0:
            n += 1
        rec = fr[: n * rs].reshape(n, rs)
        assert np.all((rec[:, 0].astype(int) | (rec[:, 1].astype(int) << 8)) == klen)
        keys.append(rec[:, 2:2 + klen].copy())
        vals.append(rec[:, 2 + klen:].copy().view(np.float64).reshape(n, width))
    if not keys:
        return np.zeros((0, klen), np.uint8), np.zeros((0, width))
    return np.concatenate(keys), np.concatenate(vals)


def sort_by_key(kb, vals):
    order = np.lexsort(kb.T[::-1]) if kb.shape[0] else np.zeros(0, int)
    return kb[order], vals[order]


def run_reference(algo, frames, agg, stats, M, p, seed):
    cfg = EngineConfig(memory_frames=M, frame_size=p, seed=seed)
    outs = []
    with OpContext(cfg, agg) as ctx:
        op = OPERATORS[algo](ctx, stats)
        src = FrameSource.from_frames(list(frames), p)
        t0 = time.perf_counter()
        for fr in run_operator(op, src):
            outs.append(np.array(fr, copy=True))
        dt = time.perf_counter() - t0
        met = ctx.metrics.as_dict()
        assert ctx.alloc.outstanding == 0
    return outs, met, dt


CASES = [
    # (case name, base config, n, overrides, [(algo, memory_frames, frame_size)])
    ("C1", "C1", 1_000_000, {}, [("hash_sort", 64, 32768), ("pre_partitioning", 64, 32768),
                                 ("original_hh", 64, 32768), ("sort_based", 64, 32768)]),
    ("C2s", "C2", 200_000, {}, [("pre_partitioning", 20, 1024), ("original_hh", 20, 1024),
                                ("hash_sort", 20, 1024), ("sort_based", 20, 1024)]),
    ("C3s05", "C3", 200_000, {"zipf_s": 0.5}, [("pre_partitioning", 256, 32768),
                                                ("hash_sort", 256, 32768)]),
    ("C3s10", "C3", 200_000, {"zipf_s": 1.0}, [("pre_partitioning", 256, 32768),
                                                ("hash_sort", 256, 32768)]),
    ("C3s15", "C3", 200_000, {"zipf_s": 1.5}, [("pre_partitioning", 256, 32768),
                                                ("hash_sort", 256, 32768)]),
    ("C4s", "C4", 40_000, {}, [("sort_based", 64, 4096), ("hash_sort", 64, 4096),
                               ("pre_partitioning", 64, 4096)]),
    ("C5s", "C5", 100_000, {"k0_range": 64, "k1_range": 16},
     [("pre_partitioning", 8, 4096), ("hash_sort", 8, 4096)]),
    ("C2tiny", "C2", 3_000, {"key_range": 500}, [("pre_partitioning", 6, 1024),
                                                 ("original_hh", 6, 1024),
                                                 ("hash_sort", 5, 1024),
                                                 ("sort_based", 5, 1024)]),
    ("C2grace", "C2", 20_000, {"key_range": 8_000}, [("pre_partitioning", 6, 1024),
                                                     ("original_hh", 6, 1024)]),
]

ENGINE_SEED = 7


def main(only=None):
    # planning / hash known answers straight from the reference
    kat = {
        "hash": [[list(b), s, int(K.hash_bytes(np.frombuffer(b, np.uint8), 0, len(b), s))]
                 for b, s in [(b"k0", 0), (b"k1", 0), (bytes(8), 0),
                              ((123456789).to_bytes(8, "big"), K.mix_seed(7, 0x22)),
                              ((2 ** 40 + 5).to_bytes(8, "big"), K.mix_seed(3, 0x111)),
                              (b"key-00000042-xxxx", 12345), (bytes(range(12)), 77)]],
        "mix_seed": [[s, t, K.mix_seed(s, t)] for s in (0, 1, 7, 2 ** 31 + 3) for t in (0x11, 0x22, 0x33, 0x45, 0x145)],
    }
    from aggbench.operators import (fallback_controller, fudge_factor, make_cuts,
                                    plan_hybrid, plan_partitions, sort_merge_levels)
    from aggbench.hash_table import plan_table
    kat["plan_partitions"] = [[g, m, plan_partitions(g, m)] for g in (0.0, 50.0, 99.0, 150.0, 1200.0, 1e9)
                              for m in (3, 10, 13, 100)]
    kat["plan_hybrid"] = []
    for g in (5.0, 40.0, 150.0, 1770.0, 1e5):
        for m in (4, 10, 13, 222, 507):
            for f in (1.0, 1.2, 1.6957):
                pl = plan_hybrid(DatasetStats(R=1e6, R_t=1e9, G=g, G_t=1e6), m, f)
                kat["plan_hybrid"].append([g, m, f, pl.P, pl.r_res, pl.r_spill, pl.grace_levels])
    kat["fudge_factor"] = [[b, e, r, bl, fudge_factor(b, e, r, bl)] for b in (26.0, 42.0, 182.0)
                           for e in (1.0, 1.2) for r in (1.0, 2.0) for bl in (False, True)]
    kat["sort_merge_levels"] = [[f, m, sort_merge_levels(f, m)] for f in (5, 100, 1e4, 1e6) for m in (3, 10, 64)]
    kat["fallback"] = [[a, b, lv, sl, fallback_controller(a, b, lv, sl)]
                       for a, b, lv, sl in [(81, 100, 1, 5), (50, 100, 1, 5), (10, 100, 6, 5), (10, 100, 5, 5)]]
    kat["make_cuts"] = [[r, P, [int(x) for x in make_cuts(r, P)]] for r, P in [(1.0, 0), (0.25, 4), (0.1, 7), (0.9, 1)]]
    kat["plan_table"] = [[nf, p, gb, sr, bl, list(plan_table(nf, p, gb, sr, bl))]
                         for nf in (2, 13, 222) for p in (1024, 32768) for gb in (26.0, 42.0)
                         for sr in (1.0,) for bl in (False, True)]
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=0)

    for name, base, n, over, runs in CASES:
        if only and name not in only:
            continue
        cfg = D.scaled(D.CONFIGS[base], n, **over)
        keys, vals = D.generate(cfg)
        agg = AggSpec.from_names(list(cfg.aggs))
        sp = ospec(cfg.aggs)
        states = init_states(sp, vals, list(cfg.bind))
        kb = D.key_bytes(keys)
        klen = kb.shape[1]
        digest = input_digest(keys, vals)
        # pin the packer against the reference codec on a prefix
        for p in sorted({r[2] for r in runs}):
            m = min(n, 3000)
            ref_frames = frames_from_records(
                [(kb[i].tobytes(), states[i].tolist()) for i in range(m)], agg.state_width, p)
            mine = pack_frames(kb[:m], states[:m], p)
            assert len(ref_frames) == len(mine) and all(
                np.array_equal(a, b) for a, b in zip(ref_frames, mine)), "packer mismatch"
        uk = np.unique(kb, axis=0)
        m_true = uk.shape[0]
        results = {}
        for algo, M, p in runs:
            frames = pack_frames(kb, states, p)
            rec_bytes = 2 + klen + 8 * agg.state_width
            stats = DatasetStats(R=max(len(frames), 1), R_t=n,
                                 G=(m_true * rec_bytes / p) if n else 0.0, G_t=m_true)
            outs, met, dt = run_reference(algo, frames, agg, stats, M, p, ENGINE_SEED)
            ok, ov = decode_fixed(outs, klen, agg.out_width)
            ok, ov = sort_by_key(ok, ov)
            assert ok.shape[0] == m_true, (name, algo, ok.shape[0], m_true)
            results[algo] = (ok, ov)
            out_path = os.path.join(HERE, f"{name}__{algo}.npz")
            meta = dict(case=name, base=base, n=n, overrides=over, seed=cfg.seed,
                        key_range=cfg.key_range, zipf_k=cfg.zipf_k, zipf_s=cfg.zipf_s,
                        k0_range=cfg.k0_range, k1_range=cfg.k1_range,
                        aggs=list(cfg.aggs), bind=list(cfg.bind), algo=algo,
                        memory_frames=M, frame_size=p, engine_seed=ENGINE_SEED,
                        stats=[stats.R, stats.R_t, stats.G, stats.G_t],
                        input_sha256=digest, metrics=met, ref_seconds=dt,
                        generator="paper_1311_0059_b200.datagen")
            np.savez_compressed(out_path, keys=ok, values=ov, meta=json.dumps(meta))
            print(f"{name:8s} {algo:18s} M={M:4d} p={p:6d} groups={ok.shape[0]:7d} "
                  f"spilled_parts={met['spilled_partitions']} depth={met['recursion_depth']} "
                  f"grace={met['grace_levels']} fb={met['fallbacks']} {dt:.2f}s", flush=True)
        # every algorithm must produce the same groups (values exact for integer data)
        algos = list(results)
        for a in algos[1:]:
            assert np.array_equal(results[a][0], results[algos[0]][0])
            d = np.abs(results[a][1] - results[algos[0]][1])
            tol = 1e-9 * np.abs(results[algos[0]][1]) + 1e-12
            assert np.all(d <= tol), (name, a, d.max())


if __name__ == "__main__":
    main(sys.argv[1:] or None)
