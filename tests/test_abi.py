"""CPU-only checks of the C ABI boundary: libpt.so loads, exports every symbol
include/pt.h declares, its host-only logic works, and the product path fails
loudly (no CPU fallback) when there is no GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2507_15277_b200 import pt


def header_functions():
    src = open(os.path.join(ROOT, "include", "pt.h")).read()
    return sorted(set(re.findall(r"^\s*(?:pt_status|void|int32_t|const char \*)\s*\**\s*(pt_\w+)\s*\(",
                                 src, flags=re.M)))


def test_header_declares_the_boundary():
    names = header_functions()
    for f in ("pt_load_perf", "pt_score_sets", "pt_greedy_select", "pt_exhaustive_best",
              "pt_eval_holdout"):
        assert f in names
    assert set(names) == set(pt.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(pt.LIB_PATH)
    for name in header_functions():
        assert hasattr(lib, name), name


def test_merge_top2_orders_by_score_then_tuple():
    rng = np.random.default_rng(0)
    for _ in range(50):
        n, k = rng.integers(1, 12), rng.integers(1, 5)
        s = rng.integers(0, 4, size=n).astype(np.float64)          # many exact ties
        s[rng.random(n) < 0.2] = np.inf                            # absent records
        t = np.sort(rng.integers(0, 6, size=(n, k)), axis=1)
        recs = sorted({(float(s[i]), tuple(int(x) for x in t[i])) for i in range(n)
                       if np.isfinite(s[i])})
        if not recs:
            with pytest.raises(pt.PTError):
                pt.pt_merge_top2(s, t, k)
            continue
        b, r, (s1, s2) = pt.pt_merge_top2(s, t, k)
        assert (s1, b) == recs[0]
        if len(recs) > 1:
            assert (s2, r) == recs[1]
        else:
            assert r is None and s2 == np.inf


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(pt.PTError) as ei:
        pt.pt_load_perf(np.ones((2, 3), np.float32))
    assert ei.value.code == pt.PT_ECUDA
