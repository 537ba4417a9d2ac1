"""Throughput of the reference-shaped operator API (frames in, frames out:
OPERATORS[algo](ctx, stats) + run_operator) on a C2-shaped input of fixed-width keys.
The frames are the reference wire format (2-byte key length, key bytes, f64 state
words); Operator.push decodes them on the host (vectorised), the columns go through
the C ABI.    python tools/frames_time.py [records] [algo]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_0059_b200.core import AggSpec, DatasetStats, pack_fixed
from paper_1311_0059_b200.operators import OPERATORS, EngineConfig, FrameSource, OpContext, run_operator

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
algo = sys.argv[2] if len(sys.argv) > 2 else "pre_partitioning"
G = n // 100
rng = np.random.default_rng(1)
keys = rng.integers(0, G, n).astype(">i8").view(np.uint8).reshape(n, 8)
v = rng.integers(0, 1000, n).astype(np.float64)
agg = AggSpec.from_names(["count", "sum", "min", "max"])
states = np.stack([np.ones(n), v, v, v], axis=1)      # init ops applied (reference state records)
fs = 32768
t0 = time.time(); fr = pack_fixed(keys, states, fs); t_pack = time.time() - t0
frames = [fr[i] for i in range(fr.shape[0])]
rec_b = 2 + 8 + 8 * 4
stats = DatasetStats(R=len(frames), R_t=n, G=G * rec_b / fs, G_t=G)
M = max(8, int(0.125 * G * rec_b / fs))                  # a budget of ~1/8 of the groups
cfg = EngineConfig(memory_frames=M, frame_size=fs, seed=3)
for it in range(2):
    t0 = time.time()
    with OpContext(cfg, agg) as ctx:
        op = OPERATORS[algo](ctx, stats)
        out = sum(1 for _ in run_operator(op, FrameSource.from_frames(frames, fs)))
        met = ctx.metrics
    dt = time.time() - t0
print(f"{algo}: {n} records in {len(frames)} frames of {fs} B (packing {t_pack:.2f} s, untimed); "
      f"open/push/close {dt*1e3:.0f} ms = {n/dt/1e6:.1f} M rec/s, {out} output frames, {met.output_groups} groups, "
      f"spilled {met.spilled_records}")
