"""The N>1 path on the CPU: world_size-2 gloo processes run the exchange
collective (paper_1311_0059_b200.exchange.exchange_records) over packed
partial-state records; merging what each rank receives must give the global
group-by, with disjoint key sets per rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partials(keys, vals):
    """Local combine (count, sum, min, max) -> AoS int64 records [key, c, s, mn, mx]."""
    u, inv = np.unique(keys, return_inverse=True)
    c = np.bincount(inv, minlength=len(u)).astype(np.int64)
    s = np.zeros(len(u), np.int64)
    np.add.at(s, inv, vals)
    mn = np.full(len(u), np.iinfo(np.int64).max)
    np.minimum.at(mn, inv, vals)
    mx = np.full(len(u), np.iinfo(np.int64).min)
    np.maximum.at(mx, inv, vals)
    return np.stack([u, c, s, mn, mx], axis=1)


def _worker(rank, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_1311_0059_b200 import datagen as D
    from paper_1311_0059_b200.exchange import exchange_records
    cfg = D.scaled(D.CONFIGS["C2"], 40_000, key_range=5_000)
    n = cfg.n // WORLD
    keys, vals = D.generate(cfg, rank * n, n)            # this rank's shard
    recs = _partials(keys[0], vals[0])
    dest = (recs[:, 0].view(np.uint64) * np.uint64(0x9E3779B97F4A7C15) >> np.uint64(63)).astype(np.int64)
    order = np.argsort(dest, kind="stable")
    packed = np.ascontiguousarray(recs[order])
    counts = np.bincount(dest, minlength=WORLD).tolist()
    send = torch.from_numpy(packed.view(np.uint8).reshape(-1).copy())
    recv, rcounts = exchange_records(send, counts, 5 * 8)
    got = recv.numpy().view(np.int64).reshape(-1, 5)
    # merge (merge ops: add, add, min, max) and finalize
    u, inv = np.unique(got[:, 0], return_inverse=True)
    merged = np.zeros((len(u), 4), np.int64)
    np.add.at(merged[:, 0], inv, got[:, 1])
    np.add.at(merged[:, 1], inv, got[:, 2])
    merged[:, 2] = np.iinfo(np.int64).max
    merged[:, 3] = np.iinfo(np.int64).min
    np.minimum.at(merged[:, 2], inv, got[:, 3])
    np.maximum.at(merged[:, 3], inv, got[:, 4])
    out_q.put((rank, u, merged, rcounts))
    dist.destroy_process_group()


def test_two_rank_exchange_gives_global_groupby():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    ukeys = [r[1] for r in res]
    assert len(np.intersect1d(ukeys[0], ukeys[1])) == 0          # disjoint key sets
    allk = np.concatenate(ukeys)
    allv = np.concatenate([r[2] for r in res]).astype(np.float64)
    order = np.argsort(allk)
    from paper_1311_0059_b200 import datagen as D
    cfg = D.scaled(D.CONFIGS["C2"], 40_000, key_range=5_000)
    keys, vals = D.generate(cfg)
    uk, want, _ = O.groupby_numpy(keys, vals, O.ospec(cfg.aggs))
    assert np.array_equal(allk[order], uk[:, 0].view(np.int64))
    assert np.array_equal(allv[order], want)
