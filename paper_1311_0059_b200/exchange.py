"""Multi-GPU group-by: local combine -> hash exchange -> merge.

One process per GPU.  Every rank aggregates its own shard with a handle that
keeps unfinalized states (``emit_partials``); ``aggb_exchange_pack`` groups
the partial groups by ``dest = hash(key, exchange seed) % world`` into one
device buffer; one all-to-all of counts and one all-to-allv of the packed
records (torch.distributed over NCCL / NVLink) move them; a merge handle of the
same spec folds what this rank received (merge ops only) and finishes.  Key
sets are disjoint across ranks after the exchange, so the job's output is the
concatenation of the ranks' outputs.  The exchange seed is independent of the
table, partition and level seeds.

When local aggregation would not shrink what is sent (C4: ~0.5N distinct
keys), ``RawExchanger`` exchanges input rows first (``aggb_exchange_pack_raw``)
and aggregates once on the receiving rank; ``choose_exchange`` picks the mode
from the group estimate.

``exchange_records`` is the collective alone (byte buffers + per-destination
record counts); it has no CUDA dependency and is tested with gloo on the CPU.
The per-destination counts are host values (the pack returns them): given a
CPU-side ``meta_group`` (gloo), they are exchanged there, so the data
all-to-allv is the only collective on the device stream and nothing waits on
the device for the counts.  Over a gloo data group (no GPU collectives: the
two-processes-on-one-GPU test, tests/test_gpu_exchange.py) CUDA buffers are
staged through host memory.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from paper_1311_0059_b200 import _native as N


def exchange_records(send: torch.Tensor, send_counts: list, record_bytes: int, group=None, meta_group=None):
    """All-to-allv of packed records.

    send: 1-D uint8 tensor, records grouped by destination rank in rank order.
    send_counts: records per destination (len == world size), host ints.
    meta_group: optional CPU (gloo) group for the counts exchange.
    Returns (recv uint8 tensor on send's device, recv_counts list).
    """
    world = dist.get_world_size(group)
    dev = send.device
    if meta_group is not None:
        sc = torch.tensor(send_counts, dtype=torch.int64)
        rc = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(rc, sc, group=meta_group)
    else:
        sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
        rc = torch.empty(world, dtype=torch.int64, device=dev)
        dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.cpu().tolist()]
    payload = send[: sum(send_counts) * record_bytes]
    stage = dev.type == "cuda" and dist.get_backend(group) == "gloo"
    if stage:  # gloo moves host memory only
        payload = payload.cpu()
    recv = torch.empty(sum(recv_counts) * record_bytes, dtype=torch.uint8, device="cpu" if stage else dev)
    dist.all_to_all_single(recv, payload,
                           output_split_sizes=[c * record_bytes for c in recv_counts],
                           input_split_sizes=[c * record_bytes for c in send_counts], group=group)
    if stage:
        recv = recv.to(dev)
    return recv, recv_counts


def expected_distinct(n_records: float, groups: float) -> float:
    """E[distinct keys] of n uniform draws over `groups` keys (an upper bound
    under skew): G (1 - exp(-n / G))."""
    import math
    if groups <= 0 or n_records <= 0:
        return 0.0
    return groups * -math.expm1(-n_records / groups)


def choose_exchange(local_records: int, group_estimate: float, raw_bytes: int, partial_bytes: int) -> str:
    """exchange raw rows when local aggregation would not
    shrink the bytes to send (local_groups x state_B >= local_records x live_B),
    partial groups otherwise.  C2: 1M x 40 B << 100M x 16 B -> partial;
    C4 at 8 GPUs: ~113M x 24 B > 125M x 16 B -> raw."""
    if local_records <= 0:
        return "partial"
    local_groups = expected_distinct(local_records, group_estimate)
    return "raw" if local_groups * partial_bytes >= local_records * raw_bytes else "partial"


class RawExchanger:
    """Raw-first exchange: pack input rows by destination, all-to-allv, then one
    aggregation of what this rank received (key sets disjoint across ranks)."""

    def __init__(self, handle, device, stream, meta_group=None):
        self.g = handle
        self.device = device
        self.stream = stream
        self.meta_group = meta_group
        self._send = None
        self.last_counts = None

    def run(self, keys, vals, group=None):
        world = dist.get_world_size(group)
        self._send, counts, rb = self.g.pack_raw(keys, vals, world, out=self._send)
        if self.stream is not None and self.device.type == "cuda":
            with torch.cuda.stream(self.stream):
                recv, recv_counts = exchange_records(self._send, counts, rb, group, self.meta_group)
        else:
            recv, recv_counts = exchange_records(self._send, counts, rb, group, self.meta_group)
        self.last_counts = (counts, recv_counts)
        self.g.reset()
        total = sum(recv_counts)
        if total:
            self.g.push_packed_raw(recv, total)
        return self.g.finish()


class Exchanger:
    """Drives the exchange + merge after a local handle has finished.

    ``local`` must be a GroupBy created with ``emit_partials=True``.  The merge
    handle has the same spec; its budget is the local one, raised to the
    partial groups this rank expects to receive (``expect_groups``: ~G / world
    over the job) so the merge aggregates in place instead of spilling again.
    """

    def __init__(self, local, agg, key_types, val_types, device, stream, rank, world, meta_group=None,
                 expect_groups=0, **kw):
        from paper_1311_0059_b200.engine import GroupBy
        self.local = local
        self.rank, self.world = rank, world
        self.device = device
        self.meta_group = meta_group
        budget = kw.pop("budget_groups", -1)
        if budget > 0 and expect_groups > 0:
            budget = max(budget, int(1.25 * expect_groups) + 1024)
        self.merge = GroupBy(local.algo if local.algo != "sort_based" else "pre_partitioning",
                             agg, key_types, val_types, device=device.index, stream=stream,
                             budget_groups=budget, **kw)
        self.rec_bytes = int(local.L.aggb_exchange_record_bytes(local.h))
        self.stream = stream
        self._send = None
        self.last_counts = None

    def run(self):
        L = self.local.L
        res = self.local._result
        n = res.n_groups
        need = max(n, 1) * self.rec_bytes
        if self._send is None or self._send.numel() < need:
            self._send = torch.empty(int(need * 1.25), dtype=torch.uint8, device=self.device)
        counts = (ctypes.c_int64 * self.world)()
        N.check(L.aggb_exchange_pack(self.local.h, self.world, ctypes.c_void_p(self._send.data_ptr()),
                                     counts), "aggb_exchange_pack")
        send_counts = [int(c) for c in counts]
        # the collectives are ordered on the handles' stream: the pack kernel
        # before them, the merge after them (NCCL waits on / signals the
        # current stream; a side stream would race the receive buffer)
        if self.stream is not None and self.device.type == "cuda":
            with torch.cuda.stream(self.stream):
                recv, recv_counts = exchange_records(self._send, send_counts, self.rec_bytes,
                                                     meta_group=self.meta_group)
        else:
            recv, recv_counts = exchange_records(self._send, send_counts, self.rec_bytes,
                                                 meta_group=self.meta_group)
        self.last_counts = (send_counts, recv_counts)
        self.merge.reset()
        total = sum(recv_counts)
        if total:
            N.check(L.aggb_push_partials(self.merge.h, ctypes.c_void_p(recv.data_ptr()), total),
                    "aggb_push_partials")
        return self.merge.finish()
