"""The C ABI: the library loads here (no GPU needed) and exports every function
include/aggb200.h declares; the Python binding maps every status onto the
reference's exception classes."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1311_0059_b200 import _native as N
from paper_1311_0059_b200 import core


def declared_functions():
    src = open(N.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(aggb_\w+)\s*\(", src, re.M)))


def test_header_declares_exports():
    assert set(declared_functions()) == set(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("libaggb200.so not built (run __graft_entry__.build())")
    L = ctypes.CDLL(N.LIB_PATH)
    for name in declared_functions():
        assert hasattr(L, name), name
    assert N.load().aggb_version().decode().startswith("aggb200")


def test_library_is_sm100a():
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("library not built")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header():
    # sizes of the POD structs as compiled by a C compiler from the header
    code = r'''
#include <stdio.h>
#include "aggb200.h"
int main(){printf("%zu %zu %zu %zu %zu\n", sizeof(aggb_config), sizeof(aggb_spec),
 sizeof(aggb_input), sizeof(aggb_result), sizeof(aggb_metrics)); return 0;}
'''
    import tempfile
    d = tempfile.mkdtemp()
    c = os.path.join(d, "s.c")
    open(c, "w").write(code)
    exe = os.path.join(d, "s")
    subprocess.check_call(["gcc", "-I", os.path.dirname(N.HEADER), c, "-o", exe])
    sizes = [int(x) for x in subprocess.check_output([exe]).split()]
    assert sizes == [ctypes.sizeof(N.Config), ctypes.sizeof(N.Spec), ctypes.sizeof(N.Input),
                     ctypes.sizeof(N.Result), ctypes.sizeof(N.Metrics)]


def test_status_to_exception_mapping(monkeypatch):
    monkeypatch.setattr(N, "last_error", lambda: "msg")
    cases = {N.AGGB_INVALID_BUDGET: core.InvalidBudget, N.AGGB_SPEC_ERROR: core.SpecError,
             N.AGGB_CAPACITY_EXCEEDED: core.CapacityExceeded,
             N.AGGB_ORDER_ERROR: core.MergeOrderError,
             N.AGGB_BUDGET_EXHAUSTED: core.BudgetExhausted,
             N.AGGB_INVALID_RECORD: core.InvalidRecord,
             N.AGGB_CUDA_ERROR: core.AggregationError}
    for st, cls in cases.items():
        with pytest.raises(cls):
            N.check(st)
    N.check(N.AGGB_OK)


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(N, "_lib", None)
    with pytest.raises(N.NativeLibraryMissing):
        N.load("/nonexistent/libaggb200.so")
