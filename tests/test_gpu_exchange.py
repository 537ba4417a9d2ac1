"""The multi-GPU path executed for real: two processes, each
with the real GroupBy on the one leased GPU, exchange over gloo (CUDA buffers
staged through host memory: gloo moves host memory; on an 8-GPU node the data
group is NCCL over NVLink, bench.py --gpus N).  Both exchange modes:

* partial: local combine (``emit_partials``), ``aggb_exchange_pack`` by
  hash(key) % world, all-to-allv, ``aggb_push_partials`` + merge (Exchanger);
* raw-first: ``aggb_exchange_pack_raw`` of the input rows, all-to-allv, one
  aggregation on the receiving rank (RawExchanger).

The counts travel over a second (CPU) group, as bench.py does.  The union of
the ranks' outputs must equal the oracle's group-by of the whole input, and
key sets must be disjoint across ranks.  No kernel of one process waits on the
other's (the collectives are host-side), so two processes can share the GPU.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(case):
    from paper_1311_0059_b200 import datagen as D
    if case == "C5":
        return D.scaled(D.CONFIGS["C5"], 400_000)
    return D.scaled(D.CONFIGS["C2"], 2_000_000, key_range=200_000)


def _worker(rank, port, mode, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        meta = dist.new_group(backend="gloo")
        import bench
        from paper_1311_0059_b200.core import DatasetStats
        from paper_1311_0059_b200.engine import GroupBy
        from paper_1311_0059_b200.exchange import Exchanger, RawExchanger
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        cfg = _cfg(case)
        n = cfg.n // WORLD
        keys, vals = bench.make_inputs(cfg, rank * n, n, dev)  # this rank's shard
        torch.cuda.synchronize()
        G = cfg.key_range or cfg.k0_range * cfg.k1_range
        st = DatasetStats(R=1, R_t=n, G=1, G_t=min(G, n))
        agg = bench.spec_of(cfg)
        kt, vt = bench.types_of(keys), bench.types_of(vals)
        budget = max(1024, min(G, n) // 8)  # forces local spill
        stream = torch.cuda.current_stream(dev)
        g = GroupBy("pre_partitioning", agg, kt, vt, budget_groups=budget, stats=st, seed=1234,
                    device=0, stream=stream, emit_partials=mode == "partial")
        if mode == "partial":
            g.push(keys, vals)
            g.finish()
            x = Exchanger(g, agg, kt, vt, dev, stream, rank, WORLD, meta_group=meta, expect_groups=min(G, cfg.n) / WORLD,
                          stats=st, seed=1234, budget_groups=budget)
            x.run()
            out = x.merge
        else:
            x = RawExchanger(g, dev, stream, meta_group=meta)
            x.run(keys, vals)
            out = g
        res = out.result()
        shard = ([k.cpu().numpy() for k in keys], [v.cpu().numpy() for v in vals])  # the bytes it aggregated
        q.put((rank, [np.asarray(k).astype(np.int64) for k in res.keys],
               [np.asarray(v) for v in res.values], x.last_counts, None, shard))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        import traceback
        q.put((rank, None, None, None, traceback.format_exc(), None))


@pytest.mark.parametrize("mode,case", [("partial", "C2"), ("raw", "C2"), ("partial", "C5")])
def test_two_processes_exchange_and_merge(mode, case):
    import torch.multiprocessing as mp
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, mode, case, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[4] is None, r[4]
    cfg = _cfg(case)
    # the whole input: both ranks' device-generated shards (C5's normal columns
    # come from the device generator; the host's libm would give other bytes)
    res.sort(key=lambda r: r[0])
    keys = [np.concatenate([r[5][0][i] for r in res]) for i in range(len(res[0][5][0]))]
    vals = [np.concatenate([r[5][1][i] for r in res]) for i in range(len(res[0][5][1]))]
    sp = O.ospec(list(cfg.aggs))
    want_k, want_v, _ = O.groupby_numpy(keys, vals, sp, list(cfg.bind))
    # disjoint key sets, union = the oracle's groups
    got_k = [np.concatenate([r[1][i] for r in res]) for i in range(len(keys))]
    got_v = np.stack([np.concatenate([np.asarray(r[2][j], np.float64) for r in res])
                      for j in range(len(cfg.aggs))], axis=1)
    order = np.lexsort(got_k[::-1])
    got_k = [k[order] for k in got_k]
    got_v = got_v[order]
    if len(keys) == 1:
        wk = [want_k[:, 0].view(np.int64)]
    else:
        wk = [want_k[:, 0].view(np.int64), want_k[:, 1].astype(np.uint32).view(np.int32).astype(np.int64)]
    assert len(got_k[0]) == len(wk[0]), "groups duplicated across ranks or missing"
    for a, b in zip(got_k, wk):
        assert np.array_equal(a, b)
    from conftest import assert_values_match, float_out_cols
    assert_values_match(got_v, want_v, float_out_cols(cfg))
    # every record was sent somewhere; both ranks received records
    sent = [sum(r[3][0]) for r in res]
    recv = [sum(r[3][1]) for r in res]
    assert sum(sent) == sum(recv) and all(x > 0 for x in recv)
