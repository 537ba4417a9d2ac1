"""Pin the CPU oracle against the reference itself (tests/golden/, made by
tests/golden/make_golden.py running /root/reference in the build container)."""

import json
import os

import numpy as np
import pytest

from conftest import (GOLDEN_DIR, assert_values_match, float_out_cols, golden_files,
                      golden_inputs, load_golden)
from oracle import oracle as O
from paper_1311_0059_b200 import datagen as D

KAT = json.load(open(os.path.join(GOLDEN_DIR, "kat.json")))


def test_hash_and_seed_known_answers():
    L = O.lib()
    for key, seed, want in KAT["hash"]:
        kb = np.array(key, np.uint8)
        assert int(O.hash_bytes(kb[None, :], seed)[0]) == want
        assert L.ora_hash_bytes(kb.ctypes.data, len(kb), seed) == want
    for s, t, want in KAT["mix_seed"]:
        assert O.mix_seed(s, t) == want
        assert L.ora_mix_seed(s, t) == want


def test_survey_appendix_a_vectors():
    cases = [(b"k0", 0, 579624470), (b"k1", 0, 2910397746), (bytes(8), 0, 2943932163),
             ((123456789).to_bytes(8, "big"), O.mix_seed(7, 0x22), 2445317540),
             ((2 ** 40 + 5).to_bytes(8, "big"), O.mix_seed(3, 0x111), 1877518074)]
    for key, seed, want in cases:
        assert int(O.hash_bytes(np.frombuffer(key, np.uint8)[None, :], seed)[0]) == want
    assert O.mix_seed(0, 0x11) == 1125321767


def test_c_port_planning_known_answers():
    import ctypes
    L = O.lib()
    for g, m, want in KAT["plan_partitions"]:
        P = ctypes.c_int32(-1)
        st = L.ora_plan_partitions(g, m, ctypes.byref(P))
        if m < 3:
            assert st == 1
        else:
            assert st == 0 and P.value == want
    for b, e, r, bl, want in KAT["fudge_factor"]:
        assert L.ora_fudge_factor(b, e, r, int(bl)) == pytest.approx(want, rel=1e-15)
    for f, m, want in KAT["sort_merge_levels"]:
        assert L.ora_sort_merge_levels(f, m) == want
    for a, b, lv, sl, want in KAT["fallback"]:
        assert L.ora_fallback(a, b, lv, sl) == (1 if want == "fallback_hash_sort" else 0)
    for r, P, want in KAT["make_cuts"]:
        out = np.zeros(max(P + 1, 1), np.int64)
        L.ora_make_cuts(r, P, out.ctypes.data)
        assert out.tolist() == want


@pytest.mark.parametrize("path", golden_files(), ids=lambda p: os.path.basename(p)[:-4])
def test_c_port_matches_reference(path):
    meta, gkeys, gvals = load_golden(path)
    cfg, keys, vals = golden_inputs(meta)
    sp = O.ospec(cfg.aggs)
    states = O.init_states(sp, vals, list(cfg.bind))
    kb = D.key_bytes(keys)
    frames = O.pack_frames(kb, states, meta["frame_size"])
    res = O.run_port(meta["algo"], frames, sp, memory_frames=meta["memory_frames"],
                     frame_size=meta["frame_size"], stats=meta["stats"],
                     seed=meta["engine_seed"], kmax=kb.shape[1])
    order = np.lexsort(res.keys.T[::-1])
    assert np.array_equal(res.keys[order], gkeys)
    assert_values_match(res.values[order], gvals, float_out_cols(cfg))
    rm = meta["metrics"]
    assert res.metrics["output_groups"] == rm["output_groups"]
    if meta["algo"] in ("pre_partitioning", "original_hh"):
        # the spill / recursion structure is restated exactly
        for k in ("spilled_partitions", "recursion_depth", "grace_levels", "fallbacks"):
            assert res.metrics[k] == rm[k], (k, res.metrics[k], rm[k])
        if rm["fallbacks"] == 0:
            assert res.metrics["high_water"] == rm["high_water"]


@pytest.mark.parametrize("path", [p for p in golden_files() if "__pre_partitioning" in p
                                  or "__sort_based" in p], ids=lambda p: os.path.basename(p)[:-4])
def test_numpy_restatement_matches_reference(path):
    meta, gkeys, gvals = load_golden(path)
    cfg, keys, vals = golden_inputs(meta)
    sp = O.ospec(cfg.aggs)
    uk, out, _ = O.groupby_numpy(keys, vals, sp, list(cfg.bind))
    kb = D.key_bytes([uk[:, i].view(np.int64) if keys[i].dtype.itemsize == 8
                      else uk[:, i].astype(np.uint32).view(np.int32) for i in range(len(keys))])
    assert np.array_equal(kb, gkeys)
    assert_values_match(out, gvals, float_out_cols(cfg))


def test_packer_round_trip():
    cfg = D.scaled(D.CONFIGS["C2"], 5000)
    keys, vals = D.generate(cfg)
    sp = O.ospec(cfg.aggs)
    st = O.init_states(sp, vals)
    fr = O.pack_frames(D.key_bytes(keys), st, 1024)
    rs = 2 + 8 + 8 * sp.state_width
    assert fr.shape[1] == 1024 and fr.shape[0] == -(-5000 // (1024 // rs))
    rec = fr[:, : (1024 // rs) * rs].reshape(-1, rs)[:5000]
    assert np.all(rec[:, 0] == 8) and np.all(rec[:, 1] == 0)
    assert np.array_equal(rec[:, 10:].copy().view(np.float64), st)
