"""Shared fixtures: the gpu marker, golden-fixture loading, input rebuilding.

Tests marked ``gpu`` need a B200 and the built CUDA library; everything else
runs on the CPU container (oracle pinning, host logic, C-ABI symbol checks,
gloo multi-process exchange).
"""

import glob
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN_DIR = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU and the built CUDA library")


def golden_files():
    return sorted(glob.glob(os.path.join(GOLDEN_DIR, "*__*.npz")))


def load_golden(path):
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    return meta, z["keys"], z["values"]


def golden_config(meta):
    from paper_1311_0059_b200 import datagen as D
    return D.scaled(D.CONFIGS[meta["base"]], meta["n"], **meta["overrides"])


def golden_inputs(meta):
    """Regenerate the golden case's inputs and check they are the same bytes."""
    import hashlib
    from paper_1311_0059_b200 import datagen as D
    cfg = golden_config(meta)
    keys, vals = D.generate(cfg)
    h = hashlib.sha256()
    for a in list(keys) + list(vals):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == meta["input_sha256"], "generator drifted from the golden inputs"
    return cfg, keys, vals


def assert_values_match(got, want, float_cols, rel=1e-9):
    """Exact for integer-derived columns; relative 1e-9 for fp64 SUM/AVG."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    for c in range(want.shape[1]):
        if c in float_cols:
            d = np.abs(got[:, c] - want[:, c])
            bad = d > rel * np.abs(want[:, c]) + 1e-300
            assert not bad.any(), (c, int(bad.sum()), float(d.max()))
        else:
            assert np.array_equal(got[:, c], want[:, c]), (c, np.flatnonzero(got[:, c] != want[:, c])[:5])


def float_out_cols(cfg):
    """Output columns whose values come from fp64 arithmetic (SUM/AVG of a
    float column).  MIN/MAX of float columns are selections: exact."""
    cols = set()
    float_val = [cfg.value == "u01"] if not cfg.wide else [False, False, True, True]
    for i, (name, b) in enumerate(zip(cfg.aggs, cfg.bind)):
        if name in ("sum", "avg") and float_val[b]:
            cols.add(i)
    return cols
