"""CPU ORACLE for the group-by hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this module, and only as
the checker or as the timed CPU baseline.  The product package
(``paper_1311_0059_b200``) never imports it.

Two restatements of the reference (``/root/reference/pkg/src/aggbench``):

* ``run_port`` — ctypes binding of ``aggoracle.c``, a plain-C restatement of the
  reference operators on the reference wire format (frames of
  ``u16 klen | key | f64 x nf`` records, core.py:1-10): chained hash table,
  FNV-1a ``hash_bytes``, budgeted frames, pre_partitioning / original_hh /
  grace / recursion / hash_sort / sort_based.  This is the ``"kind": "port"``
  CPU baseline.
* ``groupby_numpy`` — a vectorised numpy restatement of the aggregate
  semantics (core.py:68-185: init COPY/ONE, merge ADD/MIN/MAX, finish
  FIRST/DIV) over fixed-width keys, used for parity at sizes where the C port
  is slow.  Integer state is kept exactly (int64), matching the reference's
  float64 arithmetic whenever values stay below 2**53 (every BASELINE config).

Pinning: ``tests/test_oracle_golden.py`` checks both restatements against
``tests/golden/*.npz``, which ``tests/golden/make_golden.py`` produced by
importing and running the reference itself in the build container, and checks
``hash_bytes``/``mix_seed`` against SURVEY.md Appendix A's vectors.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libaggoracle.so")

M32 = 0xFFFFFFFF

# aggregate table (core.py:68-123): name -> (init ops, merge ops, finish op)
INIT_COPY, INIT_ONE = 0, 1
MERGE_ADD, MERGE_MIN, MERGE_MAX = 0, 1, 2
FINISH_FIRST, FINISH_DIV = 0, 1
AGG_TABLE = {
    "sum": ((INIT_COPY,), (MERGE_ADD,), FINISH_FIRST),
    "count": ((INIT_ONE,), (MERGE_ADD,), FINISH_FIRST),
    "avg": ((INIT_COPY, INIT_ONE), (MERGE_ADD, MERGE_ADD), FINISH_DIV),
    "min": ((INIT_COPY,), (MERGE_MIN,), FINISH_FIRST),
    "max": ((INIT_COPY,), (MERGE_MAX,), FINISH_FIRST),
}

ALGO_IDS = {"sort_based": 0, "hash_sort": 1, "original_hh": 2,
            "pre_partitioning": 5}

STATUS_NAMES = {1: "InvalidBudget", 3: "CapacityExceeded", 4: "SpecError",
                5: "MergeOrderError", 8: "NoMemory", 9: "AggregationError"}


class OracleError(Exception):
    def __init__(self, code: int):
        super().__init__(f"oracle status {code} ({STATUS_NAMES.get(code, '?')})")
        self.code = code


# ---------------------------------------------------------------------------
# hashing (_kernels.py:102-118), vectorised
# ---------------------------------------------------------------------------


def hash_bytes(keys: np.ndarray, seed: int) -> np.ndarray:
    """FNV-1a over each row of a (n, klen) uint8 array; _kernels.py:102-110."""
    keys = np.atleast_2d(np.asarray(keys, np.uint8))
    h = np.full(keys.shape[0], (0x811C9DC5 ^ (seed & M32)) & M32, np.uint64)
    for i in range(keys.shape[1]):
        h = ((h ^ keys[:, i].astype(np.uint64)) * np.uint64(0x01000193)) & np.uint64(M32)
    for _ in range(2):
        h = ((h ^ (h >> np.uint64(16))) * np.uint64(0x045D9F3B)) & np.uint64(M32)
    return (h ^ (h >> np.uint64(16))) & np.uint64(M32)


def mix_seed(seed: int, salt: int) -> int:
    """_kernels.py:113-118."""
    h = (seed * 2654435761 + salt * 40503 + 0x9E37) & M32
    h = ((h ^ (h >> 15)) * 2246822519) & M32
    h = ((h ^ (h >> 13)) * 3266489917) & M32
    return (h ^ (h >> 16)) & M32


# ---------------------------------------------------------------------------
# spec handling (core.py:126-185), restated
# ---------------------------------------------------------------------------


@dataclass
class OSpec:
    names: tuple
    init_ops: np.ndarray
    merge_ops: np.ndarray
    finish_ops: np.ndarray
    finish_src: np.ndarray

    @property
    def state_width(self) -> int:
        return len(self.merge_ops)

    @property
    def out_width(self) -> int:
        return len(self.finish_ops)


def ospec(names) -> OSpec:
    if isinstance(names, str):
        names = [s.strip() for s in names.split(",") if s.strip()]
    init, merge, fin, src = [], [], [], []
    for n in names:
        i, m, f = AGG_TABLE[n]
        src.append(len(merge))
        init += i
        merge += m
        fin.append(f)
    return OSpec(tuple(names), np.array(init, np.int8), np.array(merge, np.int8),
                 np.array(fin, np.int8), np.array(src, np.int8))


def init_states(spec: OSpec, cols: list, bind=None) -> np.ndarray:
    """(n, state_width) float64 initial states; bind[i] = value column of
    function i (the reference has one payload, core.py:165-169; multi-column
    configs build states caller-side as conftest.py:31-42 does)."""
    n = len(cols[0]) if cols else 0
    bind = bind or [0] * len(spec.names)
    out = np.empty((n, spec.state_width), np.float64)
    w = 0
    for fi, name in enumerate(spec.names):
        v = np.asarray(cols[bind[fi]], np.float64) if cols else np.zeros(0)
        for op in AGG_TABLE[name][0]:
            out[:, w] = v if op == INIT_COPY else 1.0
            w += 1
    return out


# ---------------------------------------------------------------------------
# wire format (core.py:193-265): fixed-width pack / decode
# ---------------------------------------------------------------------------


def pack_frames(keys: np.ndarray, states: np.ndarray, frame_size: int) -> np.ndarray:
    """Byte-identical to core.frames_from_records for fixed-width keys."""
    keys = np.asarray(keys, np.uint8)
    n, klen = keys.shape
    nf = states.shape[1]
    rs = 2 + klen + 8 * nf
    if rs > frame_size:
        raise ValueError("record larger than a frame")
    rpf = frame_size // rs
    nfr = -(-n // rpf) if n else 0
    frames = np.zeros((nfr, frame_size), np.uint8)
    if n == 0:
        return frames
    rec = np.zeros((nfr * rpf, rs), np.uint8)
    rec[:n, 0] = klen & 0xFF
    rec[:n, 1] = klen >> 8
    rec[:n, 2:2 + klen] = keys
    rec[:n, 2 + klen:] = np.ascontiguousarray(states, np.float64).view(np.uint8).reshape(n, 8 * nf)
    frames[:, :rpf * rs] = rec.reshape(nfr, rpf * rs)
    return frames


# ---------------------------------------------------------------------------
# the C port
# ---------------------------------------------------------------------------


class _Cfg(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int32), ("memory_frames", ctypes.c_int32),
                ("frame_size", ctypes.c_int32), ("input_sorted", ctypes.c_int32),
                ("fudge", ctypes.c_double), ("slot_ratio", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("group_estimate", ctypes.c_double),
                ("R", ctypes.c_double), ("R_t", ctypes.c_double),
                ("G", ctypes.c_double), ("G_t", ctypes.c_double)]


class _Spec(ctypes.Structure):
    _fields_ = [("nf", ctypes.c_int32), ("merge_ops", ctypes.c_int8 * 64),
                ("nout", ctypes.c_int32), ("finish_ops", ctypes.c_int8 * 64),
                ("finish_src", ctypes.c_int8 * 64)]


class _Metrics(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "output_groups", "frames_written", "frames_read", "spilled_partitions",
        "fallbacks", "grace_levels", "recursion_depth", "high_water",
        "spilled_records")]


class _Result(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("kmax", ctypes.c_int32),
                ("nout", ctypes.c_int32), ("keys", ctypes.POINTER(ctypes.c_uint8)),
                ("klens", ctypes.POINTER(ctypes.c_int32)),
                ("vals", ctypes.POINTER(ctypes.c_double))]


_lib = None


def build(force: bool = False) -> str:
    """Compile aggoracle.c with gcc (no reference sources involved)."""
    src = os.path.join(HERE, "aggoracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o",
                               LIB_PATH, src, "-lm"])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.ora_hash_bytes.restype = ctypes.c_uint32
        L.ora_hash_bytes.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32]
        L.ora_mix_seed.restype = ctypes.c_uint32
        L.ora_mix_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.ora_run.restype = ctypes.c_int
        L.ora_run.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(_Spec), ctypes.c_void_p,
                              ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(_Result),
                              ctypes.POINTER(_Metrics)]
        L.ora_result_free.argtypes = [ctypes.POINTER(_Result)]
        L.ora_fudge_factor.restype = ctypes.c_double
        L.ora_fudge_factor.argtypes = [ctypes.c_double] * 3 + [ctypes.c_int]
        L.ora_plan_partitions.restype = ctypes.c_int
        L.ora_plan_partitions.argtypes = [ctypes.c_double, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
        L.ora_sort_merge_levels.restype = ctypes.c_int
        L.ora_sort_merge_levels.argtypes = [ctypes.c_double, ctypes.c_int32]
        L.ora_fallback.restype = ctypes.c_int
        L.ora_fallback.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.ora_make_cuts.restype = None
        L.ora_make_cuts.argtypes = [ctypes.c_double, ctypes.c_int32, ctypes.c_void_p]
        _lib = L
    return _lib


@dataclass
class PortResult:
    keys: np.ndarray        # (n, kmax) uint8, zero padded
    klens: np.ndarray       # (n,) int32
    values: np.ndarray      # (n, out_width) float64
    metrics: dict


def run_port(algo: str, frames: np.ndarray, spec: OSpec, *, memory_frames: int,
             frame_size: int, stats: tuple, seed: int = 0, fudge: float = 1.2,
             slot_ratio: float = 1.0, group_estimate=None, input_sorted=False,
             kmax: int = 16) -> PortResult:
    """Run the C port of OPERATORS[algo] over reference-format frames."""
    L = lib()
    cfg = _Cfg(ALGO_IDS[algo], memory_frames, frame_size, int(input_sorted), fudge,
               slot_ratio, seed, -1.0 if group_estimate is None else float(group_estimate),
               *[float(x) for x in stats])
    sp = _Spec()
    sp.nf = spec.state_width
    sp.nout = spec.out_width
    for i, v in enumerate(spec.merge_ops):
        sp.merge_ops[i] = int(v)
    for i, (o, s) in enumerate(zip(spec.finish_ops, spec.finish_src)):
        sp.finish_ops[i] = int(o)
        sp.finish_src[i] = int(s)
    frames = np.ascontiguousarray(frames, np.uint8)
    res = _Result()
    met = _Metrics()
    st = L.ora_run(ctypes.byref(cfg), ctypes.byref(sp), frames.ctypes.data,
                   frames.shape[0] if frames.ndim == 2 else 0, kmax,
                   ctypes.byref(res), ctypes.byref(met))
    try:
        if st != 0:
            raise OracleError(st)
        n = res.n
        if n:
            keys = np.ctypeslib.as_array(res.keys, (n * kmax,)).reshape(n, kmax).copy()
            klens = np.ctypeslib.as_array(res.klens, (n,)).copy()
            vals = np.ctypeslib.as_array(res.vals, (n * spec.out_width,)).reshape(
                n, spec.out_width).copy()
        else:
            keys = np.zeros((0, kmax), np.uint8)
            klens = np.zeros(0, np.int32)
            vals = np.zeros((0, spec.out_width))
    finally:
        L.ora_result_free(ctypes.byref(res))
    return PortResult(keys, klens, vals, {f: getattr(met, f) for f, _ in _Metrics._fields_})


# ---------------------------------------------------------------------------
# numpy restatement of the aggregate semantics
# ---------------------------------------------------------------------------


def key_rows(keys: list) -> np.ndarray:
    """Combine key columns into one uint64-row structured order key.

    keys: list of integer columns (int64 / int32 / uint64).  Each column is
    encoded big-endian two's complement like the reference's byte keys, so the
    lexicographic byte order equals the lexicographic (unsigned) column order.
    """
    cols = []
    for k in keys:
        k = np.asarray(k)
        if k.dtype.itemsize == 8:
            cols.append(k.astype(np.int64).view(np.uint64))
        else:
            cols.append(k.astype(np.int32).view(np.uint32).astype(np.uint64))
    return np.stack(cols, axis=1) if len(cols) > 1 else cols[0][:, None]


def groupby_numpy(keys: list, cols: list, spec: OSpec, bind=None,
                  col_is_float=None):
    """Sorted-by-key group-by.  Returns (unique key rows (g, nk) uint64,
    finished values (g, out_width) float64, state arrays list).

    Integer columns aggregate in int64 (exact); float columns in float64.
    """
    kr = key_rows(keys)
    n = kr.shape[0]
    bind = bind or [0] * len(spec.names)
    col_is_float = col_is_float or [np.asarray(c).dtype.kind == "f" for c in cols]
    if n == 0:
        return kr[:0], np.zeros((0, spec.out_width)), []
    order = np.lexsort(kr.T[::-1])
    ks = kr[order]
    head = np.ones(n, bool)
    head[1:] = np.any(ks[1:] != ks[:-1], axis=1)
    starts = np.flatnonzero(head)
    counts = np.diff(np.append(starts, n))
    out = np.empty((len(starts), spec.out_width), np.float64)
    for fi, name in enumerate(spec.names):
        c = bind[fi]
        v = np.asarray(cols[c])[order] if cols else None
        isf = col_is_float[c] if cols else False
        if name == "count":
            out[:, fi] = counts.astype(np.float64)
            continue
        acc_t = np.float64 if isf else np.int64
        vv = v.astype(acc_t)
        if name in ("sum", "avg"):
            s = np.add.reduceat(vv, starts)
            out[:, fi] = s.astype(np.float64) if name == "sum" else s.astype(np.float64) / counts
        elif name == "min":
            out[:, fi] = np.minimum.reduceat(vv, starts).astype(np.float64)
        else:
            out[:, fi] = np.maximum.reduceat(vv, starts).astype(np.float64)
    return ks[starts], out, counts


# ---------------------------------------------------------------------------
# budget translation for the CPU baseline (hash_table.py:31-45, hybrid.py:89-132)
# ---------------------------------------------------------------------------


def frames_for_budget(target_groups: float, group_bytes: float, G_total: float,
                      frame_size: int = 32768, algo: str = "pre_partitioning",
                      fudge: float = 1.2, slot_ratio: float = 1.0) -> int:
    """Smallest memory_frames M whose resident table holds >= target_groups
    under the reference's planning (what BASELINE states as a group budget)."""
    import math
    bloom_cost = 1 if algo == "pre_partitioning" else 0
    G = G_total * group_bytes / frame_size
    for M in range(4, 1 << 20):
        F = (group_bytes + 8 + slot_ratio * (8 + bloom_cost)) * fudge / group_bytes
        gf = G * F
        P = 0 if gf <= M else max(1, min(math.ceil((gf - M) / (M - 2)), M - 2))
        frames = M - P if P >= 1 else M - 1
        bloom = algo == "pre_partitioning" and P > 1
        per = group_bytes + 8 + slot_ratio * (8 + (1 if bloom else 0))
        cap = int(frames * frame_size / per)
        if cap >= target_groups:
            return M
    raise ValueError("budget too large")


def prepare_port(algo: str, keys: list, vals: list, aggs, bind, budget_groups: int,
                 threads: int = 1, frame_size: int = 32768):
    """Shard a sample by key hash over `threads` independent operator instances
    (the reference's concurrency model) and pack each shard
    into reference frames; each shard gets budget/threads groups.  Untimed."""
    sp = ospec(aggs)
    states = init_states(sp, vals, list(bind))
    kr = key_rows(keys)
    kb = np.concatenate([kr[:, i:i + 1].astype(">u8").view(np.uint8).reshape(len(kr), 8)
                         if np.asarray(keys[i]).dtype.itemsize == 8 else
                         (kr[:, i].astype(np.uint32)).astype(">u4").view(np.uint8).reshape(len(kr), 4)
                         for i in range(len(keys))], axis=1)
    kb = np.ascontiguousarray(kb)
    h = hash_bytes(kb, 0x5eed) % np.uint64(threads) if threads > 1 else np.zeros(len(kb), np.uint64)
    rowv = kb.view(np.dtype((np.void, kb.shape[1]))).ravel()  # one opaque item per key row
    jobs = []
    for t in range(threads):
        sel = np.flatnonzero(h == t)
        g_t = len(np.unique(rowv[sel])) if len(sel) else 0
        rec = 2 + kb.shape[1] + 8 * sp.state_width
        fr = pack_frames(kb[sel], states[sel], frame_size)
        M = frames_for_budget(max(1, budget_groups / threads), rec, max(g_t, 1), frame_size, algo)
        stats = (max(fr.shape[0], 1), len(sel), g_t * rec / frame_size, g_t)
        jobs.append((fr, M, stats))
    return {"algo": algo, "sp": sp, "jobs": jobs, "kmax": kb.shape[1], "frame_size": frame_size}


def run_prepared(prep, seed: int = 7):
    """Time the C port over prepared shards, one thread per shard.
    Returns (seconds, groups, metrics of shard 0)."""
    import time
    from concurrent.futures import ThreadPoolExecutor

    def one(job):
        fr, M, stats = job
        return run_port(prep["algo"], fr, prep["sp"], memory_frames=M, frame_size=prep["frame_size"],
                        stats=stats, seed=seed, kmax=prep["kmax"])

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=len(prep["jobs"])) as ex:
        outs = list(ex.map(one, prep["jobs"]))
    dt = time.perf_counter() - t0
    return dt, sum(len(o.klens) for o in outs), outs[0].metrics


def timed_port_run(algo: str, keys: list, vals: list, aggs, bind, budget_groups: int,
                   threads: int = 1, frame_size: int = 32768, seed: int = 7):
    """prepare_port + run_prepared: (seconds, groups, metrics of shard 0);
    frame packing is excluded from the time."""
    return run_prepared(prepare_port(algo, keys, vals, aggs, bind, budget_groups, threads, frame_size), seed)
