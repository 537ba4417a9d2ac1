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


class _NumpyRawHandle:
    """Stand-in for GroupBy in the raw-first exchange (CPU): rows packed by
    destination as int64 [key, value] slots, then one group-by on receipt."""

    def __init__(self):
        self.rows = []

    def pack_raw(self, keys, vals, nranks, out=None):
        k = keys[0].numpy()
        v = vals[0].numpy()
        dest = (k.view(np.uint64) * np.uint64(0x9E3779B97F4A7C15) >> np.uint64(40)).astype(np.int64) % nranks
        order = np.argsort(dest, kind="stable")
        packed = np.stack([k[order], v[order]], axis=1)
        return (torch.from_numpy(packed.view(np.uint8).reshape(-1).copy()),
                np.bincount(dest, minlength=nranks).tolist(), 16)

    def reset(self):
        self.rows = []

    def push_packed_raw(self, buf, n):
        self.rows.append(buf.numpy().view(np.int64).reshape(-1, 2)[:n])

    def finish(self):
        r = np.concatenate(self.rows) if self.rows else np.zeros((0, 2), np.int64)
        return _partials(r[:, 0], r[:, 1])


def _raw_worker(rank, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_1311_0059_b200 import datagen as D
    from paper_1311_0059_b200.exchange import RawExchanger
    cfg = D.scaled(D.CONFIGS["C4"], 40_000)
    n = cfg.n // WORLD
    keys, vals = D.generate(cfg, rank * n, n)
    x = RawExchanger(_NumpyRawHandle(), torch.device("cpu"), None)
    res = x.run([torch.from_numpy(keys[0])], [torch.from_numpy(vals[0])])
    out_q.put((rank, res, x.last_counts))
    dist.destroy_process_group()


def test_two_rank_raw_exchange_gives_global_groupby():
    """Raw-first exchange (C4 shape) over gloo: every rank aggregates only what it
    received; the union of the ranks' groups is the global group-by."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_raw_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(WORLD)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    a, b = res[0][1], res[1][1]
    assert len(np.intersect1d(a[:, 0], b[:, 0])) == 0
    sent0, recv0 = res[0][2]
    sent1, recv1 = res[1][2]
    assert recv0[1] == sent1[0] and recv1[0] == sent0[1]
    from paper_1311_0059_b200 import datagen as D
    cfg = D.scaled(D.CONFIGS["C4"], 40_000)
    keys, vals = D.generate(cfg)
    want = _partials(keys[0], vals[0])
    got = np.concatenate([a, b])
    got = got[np.argsort(got[:, 0])]
    assert np.array_equal(got, want)
