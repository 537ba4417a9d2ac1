"""Columnar GPU group-by: the batched form of the reference operator loop.

``GroupBy`` owns one libaggb200 handle (one device, one stream) and mirrors
``Operator.open() / push() / close()`` (/root/reference/pkg/src/aggbench/
operators/base.py:126-182) over columns instead of 32 KB frames.  Inputs are
numpy arrays (host: copied H2D by the library on the handle's stream) or CUDA
torch tensors (device: used in place).  Results come back as numpy arrays or
as CUDA torch tensors.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from paper_1311_0059_b200 import _native as N
from paper_1311_0059_b200.core import AggSpec, DatasetStats, SpecError

_TYPES = {"i64": N.I64, "f64": N.F64, "i32": N.I32}
_NP = {N.I64: np.int64, N.F64: np.float64, N.I32: np.int32}


def _type_of(a) -> int:
    dt = str(getattr(a, "dtype", ""))
    if "int64" in dt:
        return N.I64
    if "float64" in dt:
        return N.F64
    if "int32" in dt:
        return N.I32
    raise SpecError(f"unsupported column dtype {dt!r} (int64 / int32 / float64)")


def _ptr_stride(a):
    """(pointer, byte stride, on_host) of a 1-D numpy array or CUDA tensor."""
    if isinstance(a, np.ndarray):
        if a.ndim != 1:
            raise SpecError("columns must be 1-D")
        return a.ctypes.data, a.strides[0], 1, a
    # torch tensor
    if a.dim() != 1:
        raise SpecError("columns must be 1-D")
    if not a.is_cuda:
        a = a.numpy()
        return a.ctypes.data, a.strides[0], 1, a
    return a.data_ptr(), a.stride(0) * a.element_size(), 0, a


@dataclass
class GroupResult:
    """Finished groups: key columns and one value column per function."""

    keys: list            # numpy arrays (typed per key column)
    values: list          # numpy arrays, int64 or float64 per function
    names: tuple
    sorted: bool = False

    @property
    def n_groups(self) -> int:
        return len(self.keys[0]) if self.keys else 0

    def as_float64(self) -> np.ndarray:
        """(n, out_width) float64 — the reference's output field type (core.py:5-9)."""
        if not self.values:
            return np.zeros((0, 0))
        return np.stack([np.asarray(v, np.float64) for v in self.values], axis=1)

    def sorted_by_key(self) -> "GroupResult":
        if self.n_groups == 0:
            return self
        cols = []
        for k in self.keys:
            k = np.asarray(k)
            cols.append(k.view(np.uint64) if k.dtype.itemsize == 8 else k.view(np.uint32))
        order = np.lexsort(cols[::-1])
        return GroupResult([np.asarray(k)[order] for k in self.keys],
                           [np.asarray(v)[order] for v in self.values], self.names, True)


class GroupBy:
    """One GPU group-by run (``OPERATORS[algo]`` behind ``run_operator``)."""

    def __init__(self, algo: str, agg: AggSpec, key_types=("i64",), val_types=("i64",), *,
                 memory_frames: int = 0, frame_size: int = 32768, budget_groups: int = -1,
                 stats: DatasetStats | None = None, seed: int = 0, fudge: float = 1.2,
                 slot_ratio: float = 1.0, group_estimate=None, input_sorted: bool = False,
                 level: int = 0, device: int = 0, stream=None, input_kind: str = "raw",
                 emit_partials: bool = False):
        self.L = N.load()
        if algo not in N.ALGO:
            raise SpecError(f"unknown algorithm {algo!r}")
        self.algo = algo
        self.agg = agg
        self.key_types = [(_TYPES[t] if isinstance(t, str) else t) for t in key_types]
        self.val_types = [(_TYPES[t] if isinstance(t, str) else t) for t in val_types]
        cfg = N.Config()
        cfg.algo = N.ALGO[algo]
        cfg.memory_frames = memory_frames
        cfg.frame_size = frame_size
        cfg.input_sorted = int(input_sorted)
        cfg.budget_groups = budget_groups
        cfg.fudge = fudge
        cfg.slot_ratio = slot_ratio
        cfg.seed = seed & ((1 << 64) - 1)
        cfg.group_estimate = -1.0 if group_estimate is None else float(group_estimate)
        if stats is not None:
            cfg.stats_R, cfg.stats_R_t, cfg.stats_G, cfg.stats_G_t = (
                float(stats.R), float(stats.R_t), float(stats.G), float(stats.G_t))
        cfg.level = level
        cfg.emit_partials = int(emit_partials)
        self.emit_partials = emit_partials
        sp = N.Spec()
        sp.n_fns = len(agg.fns)
        for i, (f, b) in enumerate(zip(agg.fns, agg.bind)):
            sp.fn[i] = N.FN[f.name]
            sp.col[i] = b
        sp.n_keys = len(self.key_types)
        for i, t in enumerate(self.key_types):
            sp.key_type[i] = t
        sp.n_vals = len(self.val_types)
        for i, t in enumerate(self.val_types):
            sp.val_type[i] = t
        sp.input_kind = N.INPUT_STATES if input_kind == "states" else N.INPUT_RAW
        if stream is None:
            # stream-ordered with the caller's torch work by default: device
            # columns produced on torch's current stream are complete before
            # this handle reads them (a private non-blocking stream would not
            # wait for them)
            import torch
            if torch.cuda.is_available():
                stream = torch.cuda.current_stream(device)
        self._stream = stream
        sptr = None
        if stream is not None:
            sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
            if sptr == 0:
                sptr = 1  # torch's default stream is the legacy stream: cudaStreamLegacy

        h = ctypes.c_void_p()
        N.check(self.L.aggb_create(device, ctypes.byref(cfg), ctypes.byref(sp),
                                   ctypes.c_void_p(sptr) if sptr else None, ctypes.byref(h)),
                "aggb_create")
        self.h = h
        self._result = None

    # -- push / finish ------------------------------------------------------

    def push(self, keys: list, vals: list) -> None:
        if len(keys) != len(self.key_types):
            raise SpecError(f"expected {len(self.key_types)} key columns")
        if len(vals) != len(self.val_types):
            raise SpecError(f"expected {len(self.val_types)} value columns")
        inp = N.Input()
        n = None
        keep = []
        host = None
        for i, (k, t) in enumerate(zip(keys, self.key_types)):
            if _type_of(k) != t:
                raise SpecError(f"key column {i} has the wrong dtype")
            p, s, oh, ref = _ptr_stride(k)
            keep.append(ref)
            inp.key[i], inp.key_stride[i] = p, s
            n = len(k) if n is None else n
            host = oh if host is None else host
            if oh != host or len(k) != n:
                raise SpecError("columns must share length and residency")
        for i, (v, t) in enumerate(zip(vals, self.val_types)):
            if _type_of(v) != t:
                raise SpecError(f"value column {i} has the wrong dtype")
            p, s, oh, ref = _ptr_stride(v)
            keep.append(ref)
            inp.val[i], inp.val_stride[i] = p, s
            if oh != host or len(v) != n:
                raise SpecError("columns must share length and residency")
        inp.n_rows = n or 0
        inp.on_host = host or 0
        N.check(self.L.aggb_push(self.h, ctypes.byref(inp)), "aggb_push")

    def push_raw(self, n_rows: int, key_ptrs, key_strides, val_ptrs, val_strides, on_host=0) -> None:
        """Pointer-level push (strided rows, e.g. C5's 64-byte records)."""
        inp = N.Input()
        inp.n_rows = n_rows
        for i, (p, s) in enumerate(zip(key_ptrs, key_strides)):
            inp.key[i], inp.key_stride[i] = p, s
        for i, (p, s) in enumerate(zip(val_ptrs, val_strides)):
            inp.val[i], inp.val_stride[i] = p, s
        inp.on_host = on_host
        N.check(self.L.aggb_push(self.h, ctypes.byref(inp)), "aggb_push")

    def push_partials(self, records, n: int) -> None:
        """Merge packed partial records (aggb_exchange_pack layout, device memory)."""
        ptr = records.data_ptr() if hasattr(records, "data_ptr") else int(records)
        N.check(self.L.aggb_push_partials(self.h, ctypes.c_void_p(ptr), n), "aggb_push_partials")

    def pack(self, nranks: int):
        """Pack this handle's partial groups by destination rank -> (uint8 tensor, counts)."""
        import torch
        res = self._result or self.finish()
        rb = int(self.L.aggb_exchange_record_bytes(self.h))
        buf = torch.empty(max(res.n_groups, 1) * rb, dtype=torch.uint8, device="cuda")
        counts = (ctypes.c_int64 * nranks)()
        N.check(self.L.aggb_exchange_pack(self.h, nranks, ctypes.c_void_p(buf.data_ptr()), counts),
                "aggb_exchange_pack")
        return buf, [int(c) for c in counts], rb

    def pack_raw(self, keys: list, vals: list, nranks: int, out=None):
        """Pack input rows (device columns) by destination rank before any
        aggregation -> (uint8 tensor, counts, record bytes); raw-first exchange."""
        import torch
        inp = N.Input()
        n = len(keys[0])
        keep = []
        for i, k in enumerate(keys):
            p, s, oh, ref = _ptr_stride(k)
            keep.append(ref)
            inp.key[i], inp.key_stride[i] = p, s
        for i, v in enumerate(vals):
            p, s, oh, ref = _ptr_stride(v)
            keep.append(ref)
            inp.val[i], inp.val_stride[i] = p, s
        inp.n_rows = n
        rb = int(self.L.aggb_exchange_raw_record_bytes(self.h))
        if out is None or out.numel() < max(n, 1) * rb:
            out = torch.empty(max(n, 1) * rb, dtype=torch.uint8, device=keys[0].device)
        counts = (ctypes.c_int64 * nranks)()
        N.check(self.L.aggb_exchange_pack_raw(self.h, ctypes.byref(inp), nranks,
                                              ctypes.c_void_p(out.data_ptr()), counts),
                "aggb_exchange_pack_raw")
        return out, [int(c) for c in counts], rb

    def push_packed_raw(self, buf, n: int) -> None:
        """Aggregate rows in the aggb_exchange_pack_raw layout (device buffer)."""
        rb = (len(self.key_types) + len(self.val_types)) * 8
        base = buf.data_ptr() if hasattr(buf, "data_ptr") else int(buf)
        nk = len(self.key_types)
        self.push_raw(n, [base + 8 * i for i in range(nk)], [rb] * nk,
                      [base + 8 * (nk + j) for j in range(len(self.val_types))], [rb] * len(self.val_types))

    def finish(self) -> N.Result:
        res = N.Result()
        N.check(self.L.aggb_finish(self.h, ctypes.byref(res)), "aggb_finish")
        self._result = res
        return res

    def result(self) -> GroupResult:
        """Finish (if needed) and copy the groups to host numpy arrays."""
        res = self._result or self.finish()
        n = res.n_groups
        keys = [np.empty(n, _NP[t]) for t in self.key_types]
        vals = [np.empty(n, np.float64 if res.out_type[j] == N.F64 else np.int64)
                for j in range(len(self.agg.fns))]
        kp = (ctypes.c_void_p * N.MAX_KEYS)(*[k.ctypes.data for k in keys])
        vp = (ctypes.c_void_p * N.MAX_FNS)(*[v.ctypes.data for v in vals])
        if n:
            N.check(self.L.aggb_copy_result(self.h, kp, vp), "aggb_copy_result")
        return GroupResult(keys, vals, self.agg.names, bool(res.sorted))

    def result_torch(self, device=None):
        """Finish (if needed) and copy the groups into CUDA torch tensors."""
        import torch
        res = self._result or self.finish()
        n = res.n_groups
        dev = device or torch.device("cuda", torch.cuda.current_device())
        tdt = {N.I64: torch.int64, N.I32: torch.int32, N.F64: torch.float64}
        keys = [torch.empty(n, dtype=tdt[t], device=dev) for t in self.key_types]
        vals = [torch.empty(n, dtype=torch.float64 if res.out_type[j] == N.F64 else torch.int64,
                            device=dev) for j in range(len(self.agg.fns))]
        kp = (ctypes.c_void_p * N.MAX_KEYS)(*[k.data_ptr() for k in keys])
        vp = (ctypes.c_void_p * N.MAX_FNS)(*[v.data_ptr() for v in vals])
        if n:
            N.check(self.L.aggb_copy_result(self.h, kp, vp), "aggb_copy_result")
        return keys, vals

    def metrics(self) -> dict:
        m = N.Metrics()
        N.check(self.L.aggb_metrics_get(self.h, ctypes.byref(m)), "aggb_metrics_get")
        d = m.as_dict()
        d["pool_host_bytes"] = int(self.L.aggb_pool_host_bytes(self.h))
        return d

    def profile(self, enable: bool = True) -> None:
        N.check(self.L.aggb_profile(self.h, int(enable)), "aggb_profile")

    def kernel_stats(self) -> dict:
        """{kernel name: (launches, total device ms)} since profile(True)."""
        out = {}
        i = 0
        while True:
            name = ctypes.c_char_p()
            n = ctypes.c_int64()
            ms = ctypes.c_double()
            if self.L.aggb_kernel_stats(self.h, i, ctypes.byref(name), ctypes.byref(n),
                                        ctypes.byref(ms)) != 0:
                break
            if n.value:
                out[name.value.decode()] = (n.value, ms.value)
            i += 1
        return out

    def reset(self) -> None:
        self._result = None
        N.check(self.L.aggb_reset(self.h), "aggb_reset")

    def close(self) -> None:
        if getattr(self, "h", None):
            self.L.aggb_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def groupby(algo: str, agg: AggSpec, keys: list, vals: list, **kw) -> GroupResult:
    """One-shot convenience: push all columns once and return host results."""
    with GroupBy(algo, agg, [_kname(k) for k in keys], [_kname(v) for v in vals], **kw) as g:
        g.push(keys, vals)
        return g.result()


def _kname(a) -> int:
    return _type_of(a)
