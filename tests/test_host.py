"""Host-side checks of the product library that need no GPU (-m "not gpu")."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "bbtc.h")).read()
    return sorted(set(re.findall(r"BBTC_API\s+[\w\s\*]+?\b(bbtc_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2009_12457_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(_lib.lib, s), s
        assert s in _lib.EXPORTS, s
    assert _lib.bbtc_version().decode().startswith("bbtc-b200")


def test_n_tasks_formula():
    import paper_2009_12457_b200 as bb
    for p in range(1, 80):
        assert bb.n_tasks(p) == p * (p + 1) * (p + 2) // 6 == math.comb(p + 2, 3)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 7, 16, 36, 64])
def test_task_index_matches_alg4_enumeration(p):
    """Library closed form vs the oracle's literal Alg. 4 loop."""
    import paper_2009_12457_b200 as bb
    tl = oracle.task_list(p)
    for idx, (i, j, k) in enumerate(tl.tolist()):
        assert bb.task_index(p, i, j, k) == idx
        assert bb.task_ijk(p, idx) == (i, j, k)


def test_task_index_rejects_bad_triples():
    import paper_2009_12457_b200 as bb
    with pytest.raises(bb.BBTCError):
        bb.task_index(3, 2, 1, 2)
    with pytest.raises(bb.BBTCError):
        bb.task_ijk(3, 10)


def test_no_cpu_fallback_without_gpu():
    """On a GPU-less host the library must fail loudly, never compute on the CPU."""
    import conftest
    if conftest.cuda_available():
        pytest.skip("GPU present")
    import paper_2009_12457_b200 as bb
    with pytest.raises(bb.BBTCError) as ei:
        bb.Context(0)
    assert ei.value.code == -6  # BBTC_ECUDA


def test_edge_ids_that_would_wrap_are_refused():
    """Non-u32 id arrays are range-checked before the cast: 2^32+5 or -2 must not
    silently become another vertex id."""
    from paper_2009_12457_b200 import _ptr
    ok = _ptr(np.array([0, 5, 0xFFFFFFFE], np.int64), np.uint32)
    assert ok[1] == 3 and list(ok[3]) == [0, 5, 0xFFFFFFFE]
    for bad in (np.array([1, 2**32 + 5], np.int64), np.array([3, -2], np.int64),
                np.array([0xFFFFFFFF], np.uint64), np.array([1.5]), ):
        with pytest.raises(OverflowError):
            _ptr(bad, np.uint32)
    assert _ptr(np.zeros(0, np.int64), np.uint32)[1] == 0
