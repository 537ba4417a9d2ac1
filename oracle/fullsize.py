"""Full-size oracle runs: the C port of the reference operators over inputs of
BASELINE.json's full sizes (test infrastructure; tests/test_gpu_fullsize.py).

The port needs reference state records (frames), which at full size do not
fit in memory at once (C5: 500M x 182 B), so the input is split by key into
disjoint shards, each shard is packed and aggregated by its own operator
instance (the reference's concurrency model: independent
operators over disjoint key sets), shards run on a thread pool (ctypes releases
the GIL), and the per-shard results are concatenated and sorted by key.

Every shard runs pre_partitioning with a budget that holds the shard's groups
(no spill): the results of the six operators are identical (pinned by
tests/test_oracle_golden.py), and the in-memory plan is the fast one.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from oracle import oracle as O


def _shard_of(keys: list, shards: int) -> np.ndarray:
    """Disjoint key sets: a multiplicative hash of the key columns."""
    h = np.asarray(keys[0]).astype(np.int64).view(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    if len(keys) > 1:
        k1 = np.asarray(keys[1]).astype(np.int64).view(np.uint64)
        h ^= (k1 + np.uint64(0x632BE59BD9B4E019)) * np.uint64(0xBF58476D1CE4E5B9)
        h ^= h >> np.uint64(29)
    return ((h >> np.uint64(40)) % np.uint64(shards)).astype(np.int32)


def _key_bytes(keys: list, sel: np.ndarray) -> np.ndarray:
    parts = []
    for k in keys:
        k = np.asarray(k)[sel]
        if k.dtype.itemsize == 8:
            parts.append(k.astype(np.int64).astype(">i8").view(np.uint8).reshape(-1, 8))
        else:
            parts.append(k.astype(np.int32).astype(">i4").view(np.uint8).reshape(-1, 4))
    return np.ascontiguousarray(np.concatenate(parts, axis=1))


def _decode_keys(res: O.PortResult, widths: list) -> list:
    out, off = [], 0
    for w in widths:
        b = np.ascontiguousarray(res.keys[:, off:off + w])
        if w == 8:
            out.append(b.view(">i8").ravel().astype(np.int64))
        else:
            out.append(b.view(">i4").ravel().astype(np.int64))
        off += w
    return out


def port_groupby(keys: list, vals: list, aggs, bind, groups: float, shards: int | None = None,
                 workers: int | None = None, frame_size: int = 32768):
    """Group-by of numpy columns through the C port, sharded by key; `groups`
    is the expected number of groups (each shard's table is planned for its
    share, +30%: a shard with more spills and recurses, with the same result).

    Returns (key columns sorted ascending (composite order), values (g, out)
    float64 in the reference's finished form)."""
    n = len(keys[0])
    workers = workers or max(1, min(16, os.cpu_count() or 1))
    sp = O.ospec(list(aggs))
    rec = 2 + sum(np.asarray(k).dtype.itemsize for k in keys) + 8 * sp.state_width
    if shards is None:  # ~2 GB of frames per shard
        shards = max(workers, int(np.ceil(n * rec / 2e9)))
    sid = _shard_of(keys, shards)
    order = np.argsort(sid, kind="stable")
    bounds = np.searchsorted(sid[order], np.arange(shards + 1))
    del sid
    widths = [np.asarray(k).dtype.itemsize for k in keys]

    def one(s):
        sel = order[bounds[s]:bounds[s + 1]]
        if len(sel) == 0:
            return [np.zeros(0, np.int64) for _ in keys], np.zeros((0, sp.out_width))
        kb = _key_bytes(keys, sel)
        states = O.init_states(sp, [np.asarray(v)[sel] for v in vals], list(bind))
        fr = O.pack_frames(kb, states, frame_size)
        del states
        g_t = int(min(len(sel), 1.3 * groups / shards + 1024))
        M = O.frames_for_budget(g_t, rec, g_t, frame_size, "pre_partitioning")
        stats = (fr.shape[0], len(sel), g_t * rec / frame_size, g_t)
        r = O.run_port("pre_partitioning", fr, sp, memory_frames=M, frame_size=frame_size,
                       stats=stats, seed=11, kmax=kb.shape[1])
        return _decode_keys(r, widths), r.values

    with ThreadPoolExecutor(max_workers=workers) as ex:
        parts = list(ex.map(one, range(shards)))
    kcols = [np.concatenate([p[0][i] for p in parts]) for i in range(len(keys))]
    vout = np.concatenate([p[1] for p in parts], axis=0)
    srt = np.lexsort(kcols[::-1])
    return [k[srt] for k in kcols], vout[srt]
