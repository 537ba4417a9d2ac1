"""The reference's operator plugin API, backed by the CUDA engine.

Mirrors /root/reference/pkg/src/aggbench/operators/base.py: ``EngineConfig``,
``OpContext``, ``Operator(ctx, stats, level)`` with ``open() / push(frame) /
close()``, ``run_operator`` and ``collect_groups`` keep their names, argument
meaning and error behaviour (InvalidBudget at open, MergeOrderError for a broken
sorted-input promise, AggregationError for duplicate output keys).

What differs is underneath: push() decodes each 32 KB frame of state records
(core.py:1-10) into columns on the host and hands them to one libaggb200
handle in batches; close() runs the GPU recursion and encodes finished frames.
Keys of up to 15 bytes travel as two 64-bit words (big-endian bytes, length in
the low byte — an injective encoding whose word order is the reference's byte
order, _kernels.py:121-131); longer keys are dictionary-encoded on the host
(SURVEY.md §8(f) f1).  There is no CPU aggregation path.
"""

from __future__ import annotations

import itertools
import os
import tempfile
import time
from dataclasses import dataclass
from typing import Iterator

import numpy as np

from paper_1311_0059_b200.core import (AggregationError, AggSpec, DEFAULT_FRAME_SIZE,
                                       DatasetStats, FIELD_SIZE, InvalidBudget, KLEN_SIZE,
                                       MergeOrderError, Metrics, iter_records, pack_fixed,
                                       unpack_fixed, unpack_fixed_batch)

_ctx_seq = itertools.count()

# flush decoded frames to the GPU in batches of at least this many records
PUSH_BATCH = 1 << 20
RAW_BATCH = 256  # frames decoded together by the operator API (fixed-width keys)


@dataclass
class EngineConfig:
    """Knobs shared by every operator and the planner (base.py:50-65)."""

    memory_frames: int
    frame_size: int = DEFAULT_FRAME_SIZE
    fudge: float = 1.2
    slot_ratio: float = 1.0
    seed: int = 0
    tmp_dir: str | None = None
    input_sorted: bool = False
    group_estimate: float | None = None
    # GPU additions
    device: int = 0
    budget_groups: int = 0      # >0: resident capacity in groups (overrides frames)

    def resolve_tmp(self) -> str:
        return self.tmp_dir or os.environ.get("AGGBENCH_TMP") or tempfile.gettempdir()


class FrameAllocatorView:
    """What tests read from ctx.alloc (core.py:273-331): frames outstanding and
    the high-water mark.  On the GPU the budget-governed memory is the resident
    table: an open operator holds its frames until close (outstanding), and the
    high-water mark is the frames its resident groups occupy in the reference's
    layout (record + chain link + slot, hash_table.py:31-45) plus the output
    frame, from the groups the device actually held (aggb_metrics
    resident_groups).  The device's own bytes are Metrics.device_bytes."""

    def __init__(self, budget: int):
        self.budget = budget
        self.high_water = 0
        self.outstanding = 0

    def hold(self, frames: int) -> None:
        self.outstanding += frames

    def release(self, frames: int) -> None:
        self.outstanding -= frames


class OpContext:
    """Per-run bundle: config, AggSpec, metrics, observers (base.py:68-123)."""

    def __init__(self, cfg: EngineConfig, agg: AggSpec):
        if cfg.memory_frames < 2 and cfg.budget_groups <= 0:
            raise InvalidBudget(f"need at least 2 frames, got {cfg.memory_frames}")
        self.cfg = cfg
        self.agg = agg
        self.alloc = FrameAllocatorView(cfg.memory_frames)
        self.metrics = Metrics()
        self.observers: dict = {}
        self._seq = next(_ctx_seq)

    @property
    def memory_frames(self) -> int:
        return self.cfg.memory_frames

    @property
    def frame_size(self) -> int:
        return self.cfg.frame_size

    def notify(self, event: str, *args) -> None:
        cb = self.observers.get(event)
        if cb is not None:
            cb(*args)

    def cleanup(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.cleanup()


# ---------------------------------------------------------------------------
# key <-> word encoding
# ---------------------------------------------------------------------------

MAX_WORD_KEY = 15


def encode_keys(kb: np.ndarray, klen: int) -> tuple:
    """(n, klen) uint8 keys, klen <= 15 -> (word0, word1) int64 columns."""
    n = kb.shape[0]
    pad = np.zeros((n, 16), np.uint8)
    pad[:, :klen] = kb
    pad[:, 15] = klen
    w = pad.view(">u8").reshape(n, 2).astype(np.uint64)
    return w[:, 0].view(np.int64).copy(), w[:, 1].view(np.int64).copy()


def decode_keys(w0: np.ndarray, w1: np.ndarray) -> list:
    """Inverse of encode_keys -> list of bytes."""
    n = len(w0)
    words = np.stack([np.asarray(w0).view(np.uint64), np.asarray(w1).view(np.uint64)], axis=1)
    raw = words.astype(">u8").view(np.uint8).reshape(n, 16)
    lens = raw[:, 15].astype(np.int64)
    return [bytes(raw[i, :lens[i]]) for i in range(n)]


class Operator:
    """GPU-backed operator with the reference's open / push / close protocol."""

    algo_id = "?"

    def __init__(self, ctx: OpContext, stats: DatasetStats, level: int = 0):
        self.ctx = ctx
        self.stats = stats
        self.level = level
        self.metrics = ctx.metrics
        ctx.metrics.recursion_depth = max(ctx.metrics.recursion_depth, level)
        self._engine = None
        self._raw: list = []                # frames waiting for their batch decode
        self._buf_w0: list = []
        self._buf_w1: list = []
        self._buf_st: list = []
        self._buffered = 0
        self._dict: dict | None = None      # bytes -> id for keys longer than 15 bytes
        self._dict_keys: list = []
        self._last_key = None               # sorted-input check
        self._klen_max = 0                  # widest key seen
        self._key_total = 0                 # key bytes / records pushed (high-water accounting)
        self._key_records = 0
        self._pushed_any = False
        self._opened = False

    # -- interface ----------------------------------------------------------

    def open(self) -> None:
        """Validate the budget (InvalidBudget) and create the GPU handle."""
        self._engine = self._make_engine(self.stats)
        self.ctx.alloc.hold(1)  # the handle (released by close; run_operator checks for leaks)
        self._opened = True

    def _make_engine(self, stats):
        from paper_1311_0059_b200.engine import GroupBy
        cfg = self.ctx.cfg
        agg = self.ctx.agg
        # the GPU takes reference state records: one f64 column per state field
        return GroupBy(
            self.algo_id, agg, ("i64", "i64"), ("f64",) * agg.state_width,
            memory_frames=cfg.memory_frames, frame_size=cfg.frame_size,
            budget_groups=cfg.budget_groups if cfg.budget_groups > 0 else 0,
            stats=stats, seed=cfg.seed, fudge=cfg.fudge, slot_ratio=cfg.slot_ratio,
            group_estimate=cfg.group_estimate, input_sorted=cfg.input_sorted,
            level=self.level, device=cfg.device, input_kind="states")

    def _key_bytes_seen(self, klen: int) -> None:
        """The table's capacity in groups is planned from the stats' group bytes
        (core.py DatasetStats, as the reference plans); its frames hold the actual
        records.  When the first keys are wider than the stats assumed (the
        reference's table would run out of frames earlier: first-fit failure,
        hash_table.py:40, :56-59), the handle is re-planned with the record size
        seen, before it holds anything."""
        self._klen_max = max(self._klen_max, klen)
        st, fs = self.stats, self.ctx.cfg.frame_size
        if self._pushed_any or self.ctx.cfg.budget_groups > 0 or not st.G_t or not st.G:
            return
        rec = 2 + klen + 8 * self.ctx.agg.state_width
        if rec > 1.1 * st.G * fs / st.G_t:
            self._engine.close()
            from paper_1311_0059_b200.core import DatasetStats
            self._engine = self._make_engine(DatasetStats(R=st.R, R_t=st.R_t, G=st.G_t * rec / fs, G_t=st.G_t))

    def push(self, frame: np.ndarray) -> Iterator[np.ndarray] | None:
        if not self._opened:
            self.open()
        # Frames of fixed-width keys are kept (copied: the caller may reuse its frame,
        # base.py:6-8) and decoded RAW_BATCH at a time with one reshape; a Python decode
        # per 32 KB frame held the frames-in path at 10 M records/s (tools/frames_time.py).
        if not self.ctx.cfg.input_sorted and self._dict is None:
            self._raw.append(np.array(frame, np.uint8, copy=True))
            if len(self._raw) >= RAW_BATCH:
                self._drain_raw()
            return None
        self._drain_raw()
        return self._push_one(frame)

    def _drain_raw(self) -> None:
        frames, self._raw = self._raw, []
        if not frames:
            return
        sw = self.ctx.agg.state_width
        dec = unpack_fixed_batch(frames, sw)
        if dec is None or dec[0].shape[1] > MAX_WORD_KEY:
            for f in frames:  # mixed key lengths / long keys: frame by frame
                self._push_one(f)
            return
        kb, st = dec
        if kb.shape[0]:
            self._key_bytes_seen(int(kb.shape[1]))
            self._key_total += int(kb.shape[0]) * int(kb.shape[1])
            self._key_records += int(kb.shape[0])
            w0, w1 = encode_keys(kb, kb.shape[1])
            self._buffer(w0, w1, st)
            if self._buffered >= PUSH_BATCH:
                self._flush()

    def _push_one(self, frame: np.ndarray) -> None:
        sw = self.ctx.agg.state_width
        dec = unpack_fixed([frame], sw)
        if dec is not None and dec[0].shape[0]:
            self._key_bytes_seen(int(dec[0].shape[1]))
            self._key_total += int(dec[0].shape[0]) * int(dec[0].shape[1])
            self._key_records += int(dec[0].shape[0])
        if dec is not None and dec[0].shape[1] <= MAX_WORD_KEY and self._dict is None:
            kb, st = dec
            if kb.shape[0]:
                if self.ctx.cfg.input_sorted:
                    self._check_sorted([bytes(k) for k in kb])
                w0, w1 = encode_keys(kb, kb.shape[1])
                self._buffer(w0, w1, st)
        else:
            recs = list(iter_records(np.asarray(frame, np.uint8), sw))
            if recs:
                keys = [k for k, _ in recs]
                self._key_bytes_seen(max(len(k) for k in keys))
                self._key_total += sum(len(k) for k in keys)
                self._key_records += len(keys)
                if self.ctx.cfg.input_sorted:
                    self._check_sorted(keys)
                st = np.array([v for _, v in recs], np.float64).reshape(len(recs), sw)
                w0, w1 = self._encode_var(keys)
                self._buffer(w0, w1, st)
        if self._buffered >= PUSH_BATCH:
            self._flush()
        return None

    def close(self) -> Iterator[np.ndarray]:
        if not self._opened:
            self.open()
        self._drain_raw()
        self._flush()
        res = self._engine.result()
        met = self._engine.metrics()
        m = self.metrics
        m.output_groups += res.n_groups
        m.spilled_partitions += met["spilled_partitions"]
        m.recursion_depth = max(m.recursion_depth, self.level + met["recursion_depth"])
        m.spilled_records += met["spilled_records"]
        m.spilled_bytes += met["spilled_bytes"]
        m.resident_groups += met["resident_groups"]
        m.kernel_launches += met["kernel_launches"]
        cfg = self.ctx.cfg
        klen = self._key_total / self._key_records if self._key_records else 8.0
        per = 2 + klen + 8 * self.ctx.agg.state_width + 8 + cfg.slot_ratio * 8
        frames = -(-int(met["resident_groups"] * per) // cfg.frame_size) + 1
        self.ctx.alloc.high_water = max(self.ctx.alloc.high_water, frames)
        m.high_water = max(m.high_water, self.ctx.alloc.high_water)
        m.device_bytes = max(m.device_bytes, met["high_water_bytes"])
        keys = self._decode(res.keys[0], res.keys[1])
        vals = res.as_float64()
        self._engine.close()
        self._engine = None
        self.ctx.alloc.release(1)
        if self.algo_id == "sort_based" or res.sorted:
            order = sorted(range(len(keys)), key=keys.__getitem__)
            keys = [keys[i] for i in order]
            vals = vals[order]
        yield from encode_frames(keys, vals, self.ctx.frame_size)

    # -- helpers --------------------------------------------------------------

    def _check_sorted(self, keys: list) -> None:
        prev = self._last_key
        for k in keys:
            if prev is not None and k < prev:
                raise MergeOrderError("input declared sorted but a key decreased")
            prev = k
        self._last_key = prev

    def _encode_var(self, keys: list) -> tuple:
        long = self._dict is not None or any(len(k) > MAX_WORD_KEY for k in keys)
        if not long:
            lens = {len(k) for k in keys}
            w0 = np.empty(len(keys), np.int64)
            w1 = np.empty(len(keys), np.int64)
            for L in lens:
                idx = [i for i, k in enumerate(keys) if len(k) == L]
                kb = np.frombuffer(b"".join(keys[i] for i in idx), np.uint8).reshape(len(idx), L)
                a, b = encode_keys(kb, L)
                w0[idx] = a
                w1[idx] = b
            return w0, w1
        if self._dict is None:
            if self._buffered or self._engine_pushed():
                raise AggregationError("keys longer than 15 bytes after word-encoded keys")
            self._dict = {}
        ids = np.empty(len(keys), np.int64)
        for i, k in enumerate(keys):
            v = self._dict.get(k)
            if v is None:
                v = len(self._dict_keys)
                self._dict[k] = v
                self._dict_keys.append(k)
            ids[i] = v
        return ids, np.full(len(keys), -1, np.int64)

    def _engine_pushed(self) -> bool:
        return getattr(self, "_pushed_any", False)

    def _decode(self, w0, w1) -> list:
        if self._dict is not None:
            return [self._dict_keys[int(i)] for i in w0]
        return decode_keys(w0, w1)

    def _buffer(self, w0, w1, st) -> None:
        self._buf_w0.append(w0)
        self._buf_w1.append(w1)
        self._buf_st.append(st)
        self._buffered += len(w0)

    def _flush(self) -> None:
        if not self._buffered:
            return
        w0 = np.concatenate(self._buf_w0)
        w1 = np.concatenate(self._buf_w1)
        st = np.concatenate(self._buf_st)
        cols = [np.ascontiguousarray(st[:, j]) for j in range(st.shape[1])]
        self._engine.push([w0, w1], cols)
        self._pushed_any = True
        self._buf_w0, self._buf_w1, self._buf_st = [], [], []
        self._buffered = 0


def encode_frames(keys: list, vals: np.ndarray, frame_size: int) -> Iterator[np.ndarray]:
    """Finished groups -> output frames (records never straddle frames)."""
    n = len(keys)
    if n == 0:
        return
    lens = {len(k) for k in keys}
    if len(lens) == 1:
        L = lens.pop()
        kb = np.frombuffer(b"".join(keys), np.uint8).reshape(n, L)
        for fr in pack_fixed(kb, vals, frame_size):
            yield fr
        return
    width = vals.shape[1]
    cur = np.zeros(frame_size, np.uint8)
    used = 0
    for k, v in zip(keys, vals):
        need = KLEN_SIZE + len(k) + FIELD_SIZE * width
        if used + need > frame_size:
            yield cur
            cur = np.zeros(frame_size, np.uint8)
            used = 0
        cur[used] = len(k) & 0xFF
        cur[used + 1] = len(k) >> 8
        cur[used + 2:used + 2 + len(k)] = np.frombuffer(k, np.uint8)
        cur[used + 2 + len(k):used + need].view(np.float64)[:] = v
        used += need
    if used:
        yield cur


def run_operator(op: Operator, source) -> Iterator[np.ndarray]:
    """Drive an operator over a frame source (base.py:185-217)."""
    m = op.metrics
    t0 = time.perf_counter()
    op.open()

    def finished(frames):
        for fr in frames:
            if m.time_to_first_result == 0.0:
                m.time_to_first_result = time.perf_counter() - t0
            m.frames_written_total += 1
            yield fr

    for frame in source:
        out = op.push(frame)
        if out is not None:
            yield from finished(out)
    yield from finished(op.close())
    m.frames_read_total += getattr(source, "frames_read", 0)
    m.high_water = max(m.high_water, op.ctx.alloc.high_water)
    if op.ctx.alloc.outstanding != 0:  # base.py:210-217
        raise AggregationError(f"operator leaked {op.ctx.alloc.outstanding} frame(s)")
    m.total_time = time.perf_counter() - t0


def collect_groups(op: Operator, source) -> dict:
    """Drain an operator into {key: finished values} (base.py:220-231)."""
    width = op.ctx.agg.out_width
    out: dict = {}
    for frame in run_operator(op, source):
        for key, vals in iter_records(frame, width):
            if key in out:
                raise AggregationError(f"duplicate output key {key!r}")
            out[key] = vals
    return out


class FrameSource:
    """In-memory frame source (run_store.py:134-214 FrameSource.from_frames)."""

    def __init__(self, frames, frame_size: int):
        self._frames = list(frames)
        self.frame_size = frame_size
        self.frames_read = 0
        from paper_1311_0059_b200.core import InvalidRecord
        for f in self._frames:
            if len(f) != frame_size:
                raise InvalidRecord(f"frame of {len(f)} bytes fed to a {frame_size}-byte frame source")

    @staticmethod
    def from_frames(frames, frame_size: int) -> "FrameSource":
        return FrameSource(frames, frame_size)

    def __iter__(self):
        for f in self._frames:
            yield f
