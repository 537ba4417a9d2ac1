"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference ships no data generator (SPEC.md:462-505 declares a ``datagen``
module that does not exist), and BASELINE.json names no public
dataset, so these seeded counter-based generators *are* the benchmark inputs
(SURVEY.md §8(d)).  Every value is a pure function of (seed, stream, record
index): ``x = splitmix64(base(seed, stream) + (i + 1) * GOLDEN)``.  The same
formula runs on the device (``aggb_generate``, ``k_gen`` in csrc/kernels.cuh), so
any rank can regenerate its own slice, and integer columns are bit-identical between host and device.
Normal draws go through libm on each side; parity tests for those columns copy
the device bytes back instead of regenerating them.

Draw rules: integers ``lo + x % range``; U[0,1) doubles ``(x >> 11) * 2**-53``;
normals Box-Muller; Zipf ranks by inverse CDF over a host-built fp64 table;
Zipf key ids permuted by an affine bijection of [0, K).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1

# stream ids (shared with csrc/datagen.cu)
S_KEY, S_VAL, S_K1, S_V0, S_V1, S_V2, S_V3 = 1, 2, 3, 4, 5, 6, 7
S_NORMAL_B = 100  # second uniform of a Box-Muller pair: stream + 100


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def stream_base(seed: int, stream: int) -> int:
    z = np.array([(seed * GOLDEN + stream * 0xD1B54A32D192ED03) & M64], np.uint64)
    return int(_mix64(z)[0])


def raw_u64(seed: int, stream: int, start: int, n: int) -> np.ndarray:
    """x_i for i in [start, start + n)."""
    base = np.uint64(stream_base(seed, stream))
    i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix64(base + i * np.uint64(GOLDEN))


def uniform_int(seed, stream, start, n, lo, rng) -> np.ndarray:
    return (raw_u64(seed, stream, start, n) % np.uint64(rng)).astype(np.int64) + lo


def uniform_f64(seed, stream, start, n) -> np.ndarray:
    return (raw_u64(seed, stream, start, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def normal_f64(seed, stream, start, n) -> np.ndarray:
    u1 = ((raw_u64(seed, stream, start, n) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (raw_u64(seed, stream + S_NORMAL_B, start, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def zipf_cdf(K: int, s: float) -> np.ndarray:
    w = np.arange(1, K + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    c /= c[-1]
    c[-1] = 1.0
    return c


def zipf_perm_params(K: int, seed: int) -> tuple[int, int]:
    """Affine bijection a*r + b mod K with gcd(a, K) == 1."""
    import math
    a = (stream_base(seed, 99) % K) | 1
    while math.gcd(a, K) != 1:
        a += 2
    b = stream_base(seed, 98) % K
    return a, b


def zipf_keys(seed, start, n, K, s, cdf=None) -> np.ndarray:
    cdf = zipf_cdf(K, s) if cdf is None else cdf
    u = uniform_f64(seed, S_KEY, start, n)
    rank = np.searchsorted(cdf, u, side="right")          # 0-based rank
    rank = np.minimum(rank, K - 1)
    a, b = zipf_perm_params(K, seed)
    return ((rank.astype(np.uint64) * np.uint64(a) + np.uint64(b)) % np.uint64(K)).astype(np.int64)


# ---------------------------------------------------------------------------
# the five configurations (BASELINE.json "configs")
# ---------------------------------------------------------------------------


@dataclass
class Config:
    name: str
    n: int                       # records
    seed: int
    aggs: tuple                  # reference AggSpec names
    bind: tuple                  # value column per aggregate
    key_range: int = 0           # uniform keys: U{0..key_range-1}
    zipf_k: int = 0              # zipf keys over [0, zipf_k)
    zipf_s: float = 0.0
    value: str = "int1000"       # int1000 | u01 | wide
    budget_groups: int = 0       # 0: in-memory
    algos: tuple = ("pre_partitioning",)
    wide: bool = False           # C5: 2 key columns, 4 value columns, 64-B rows
    k0_range: int = 4096
    k1_range: int = 1024
    extra: dict = field(default_factory=dict)

    @property
    def n_keys(self) -> int:
        return 2 if self.wide else 1

    @property
    def n_values(self) -> int:
        return 4 if self.wide else 1


C5_AGGS = ("count",) + ("sum", "min", "max", "avg") * 4
C5_BIND = (0,) + tuple(c for c in range(4) for _ in range(4))

CONFIGS = {
    "C1": Config("C1", 1_000_000, 1, ("count", "sum"), (0, 0), key_range=10_000,
                 algos=("hash_sort", "pre_partitioning")),
    "C2": Config("C2", 100_000_000, 2, ("count", "sum", "min", "max"), (0, 0, 0, 0),
                 key_range=1_000_000, budget_groups=125_000,
                 algos=("pre_partitioning", "original_hh")),
    "C3": Config("C3", 200_000_000, 3, ("count", "sum", "avg"), (0, 0, 0),
                 zipf_k=10_000_000, zipf_s=1.0, value="u01",
                 algos=("pre_partitioning", "hash_sort")),
    "C4": Config("C4", 1_000_000_000, 4, ("count", "sum"), (0, 0), key_range=627_500_000,
                 algos=("sort_based", "hash_sort")),
    "C5": Config("C5", 500_000_000, 5, C5_AGGS, C5_BIND, value="wide", wide=True,
                 budget_groups=83_886, algos=("pre_partitioning", "hash_sort")),
}


def scaled(cfg: Config, n: int, **over) -> Config:
    """Same shape at n records: key universes and budgets keep their ratios."""
    import dataclasses
    f = n / cfg.n
    kw = dict(n=n)
    if cfg.key_range:
        kw["key_range"] = max(1, int(round(cfg.key_range * f)))
    if cfg.zipf_k:
        kw["zipf_k"] = max(1, int(round(cfg.zipf_k * f)))
    if cfg.budget_groups and (cfg.key_range or cfg.zipf_k):
        # the budget keeps its ratio to the groups: it scales with a key universe
        # that scales (C2); C5's composite key universe (4096 x 1024) is fixed, so
        # its 2%-of-groups budget is too
        kw["budget_groups"] = max(1, int(round(cfg.budget_groups * f)))
    kw.update(over)
    return dataclasses.replace(cfg, **kw)


def generate(cfg: Config, start: int = 0, n: int | None = None):
    """Host columns for records [start, start+n): (keys list, values list)."""
    n = cfg.n - start if n is None else n
    if cfg.wide:
        k0 = uniform_int(cfg.seed, S_KEY, start, n, 0, cfg.k0_range)
        k1 = uniform_int(cfg.seed, S_K1, start, n, 0, cfg.k1_range).astype(np.int32)
        v0 = uniform_int(cfg.seed, S_V0, start, n, 0, 1 << 20)
        v1 = uniform_int(cfg.seed, S_V1, start, n, 0, 1 << 20)
        v2 = normal_f64(cfg.seed, S_V2, start, n)
        v3 = normal_f64(cfg.seed, S_V3, start, n)
        return [k0, k1], [v0, v1, v2, v3]
    if cfg.zipf_k:
        keys = zipf_keys(cfg.seed, start, n, cfg.zipf_k, cfg.zipf_s)
    else:
        keys = uniform_int(cfg.seed, S_KEY, start, n, 0, cfg.key_range)
    if cfg.value == "u01":
        vals = uniform_f64(cfg.seed, S_VAL, start, n)
    else:
        vals = uniform_int(cfg.seed, S_VAL, start, n, 0, 1000)
    return [keys], [vals]


def key_bytes(keys: list) -> np.ndarray:
    """Reference byte keys: big-endian two's complement per column
    (BE makes byte order equal numeric order for keys >= 0)."""
    parts = []
    for k in keys:
        k = np.asarray(k)
        dt = ">i8" if k.dtype.itemsize == 8 else ">i4"
        parts.append(k.astype(dt).view(np.uint8).reshape(len(k), -1))
    return np.concatenate(parts, axis=1) if parts else np.zeros((0, 0), np.uint8)


def wide_rows(keys: list, vals: list) -> np.ndarray:
    """C5 64-byte row layout: k0 i64 | k1 i32 | pad4 | v0 v1 i64 | v2 v3 f64 | pad16."""
    n = len(keys[0])
    rows = np.zeros((n, 64), np.uint8)
    rows[:, 0:8] = np.asarray(keys[0], np.int64).view(np.uint8).reshape(n, 8)
    rows[:, 8:12] = np.asarray(keys[1], np.int32).view(np.uint8).reshape(n, 4)
    for c in range(4):
        dt = np.int64 if c < 2 else np.float64
        rows[:, 16 + 8 * c:24 + 8 * c] = np.asarray(vals[c], dt).view(np.uint8).reshape(n, 8)
    return rows
